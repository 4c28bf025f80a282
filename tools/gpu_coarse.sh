#!/bin/bash
# coarse-space checks: tests, then sizes on c3 / c5 / c4 and G=1
cd $GRAFT_REPO_ROOT
python paper_2312_08201_b200/build.py > gpurun_out/co3_build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x -k "two_level or qlin or full_batch" > gpurun_out/co3_pytest.log 2>&1
B="python bench.py --no-cpu-baseline --no-e2e --steps 2 --warmup 3"
for p in 48 96 160; do timeout 600 $B --config c3 --coarse $p > gpurun_out/co3_c3_p$p.log 2>&1; done
for p in 48; do timeout 600 $B --config c5 --coarse $p > gpurun_out/co3_c5_p$p.log 2>&1; done
LYAP_GROUPS=1 timeout 600 $B --config c5 --coarse 48 > gpurun_out/co3_c5_p48_G1.log 2>&1
for p in 32 48; do timeout 600 $B --config c4 --coarse $p > gpurun_out/co3_c4_p$p.log 2>&1; done
timeout 600 $B --config c2 --coarse 32 > gpurun_out/co3_c2_p32.log 2>&1
