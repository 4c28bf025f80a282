#!/bin/bash
# coarse-space checks: tests, then sizes on c3 / c5 / c4 / c2
cd $GRAFT_REPO_ROOT
python paper_2312_08201_b200/build.py > gpurun_out/co4_build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x -k "two_level or qlin or full_batch" > gpurun_out/co4_pytest.log 2>&1
B="python bench.py --no-cpu-baseline --no-e2e --steps 2 --warmup 3"
for p in 32 48 96 160; do timeout 600 $B --config c3 --coarse $p > gpurun_out/co4_c3_p$p.log 2>&1; done
for p in 48 96; do timeout 600 $B --config c5 --coarse $p > gpurun_out/co4_c5_p$p.log 2>&1; done
for p in 32 48 96; do timeout 600 $B --config c4 --coarse $p > gpurun_out/co4_c4_p$p.log 2>&1; done
for p in 16 32; do timeout 600 $B --config c2 --coarse $p > gpurun_out/co4_c2_p$p.log 2>&1; done
