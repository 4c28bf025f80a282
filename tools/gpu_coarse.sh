#!/bin/bash
cd $GRAFT_REPO_ROOT
python paper_2312_08201_b200/build.py > gpurun_out/co9_build.log 2>&1
B="python bench.py --no-cpu-baseline --no-e2e --steps 3 --warmup 3 --config c2"
timeout 600 $B --coarse 32 > gpurun_out/co9_c2_p32.log 2>&1
timeout 600 $B --coarse 32 --no-profile > gpurun_out/co9_c2_p32_np.log 2>&1
timeout 600 $B --coarse 16 > gpurun_out/co9_c2_p16.log 2>&1
timeout 600 $B --coarse 24 > gpurun_out/co9_c2_p24.log 2>&1
timeout 600 $B --coarse 0 > gpurun_out/co9_c2_p0.log 2>&1
