#!/bin/bash
# coarse-space size sweep of the two-level preconditioner
cd $GRAFT_REPO_ROOT
python paper_2312_08201_b200/build.py > gpurun_out/co_build.log 2>&1
B="python bench.py --no-cpu-baseline --no-e2e --steps 2 --warmup 3"
for p in 32 48 96; do timeout 600 $B --config c5 --coarse $p > gpurun_out/co2_c5_p$p.log 2>&1; done
for p in 32 48 96; do timeout 600 $B --config c4 --coarse $p > gpurun_out/co2_c4_p$p.log 2>&1; done
for p in 0 32 64; do timeout 600 $B --config c2 --coarse $p > gpurun_out/co2_c2_p$p.log 2>&1; done
for p in 0 32; do timeout 600 $B --config c3 --coarse $p > gpurun_out/co2_c3_p$p.log 2>&1; done
