#!/bin/bash
cd $GRAFT_REPO_ROOT
python paper_2312_08201_b200/build.py > gpurun_out/co7_build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x -k "two_level or full_batch" > gpurun_out/co7_pytest.log 2>&1
B="python bench.py --no-cpu-baseline --no-e2e --steps 3 --warmup 3"
for c in c2 c3 c4 c5; do timeout 600 $B --config $c --coarse 32 > gpurun_out/co7_${c}_p32.log 2>&1; done
timeout 600 $B --config c2 --coarse 16 > gpurun_out/co7_c2_p16.log 2>&1
