#!/bin/bash
# coarse pipeline: benches and ncu launch lists (c2 / c3 / c5)
cd $GRAFT_REPO_ROOT
python paper_2312_08201_b200/build.py > gpurun_out/co5_build.log 2>&1
B="python bench.py --no-cpu-baseline --no-e2e --steps 2 --warmup 3"
for p in 32; do timeout 600 $B --config c2 --coarse $p > gpurun_out/co5_c2_p$p.log 2>&1; done
for p in 32 48; do timeout 600 $B --config c3 --coarse $p > gpurun_out/co5_c3_p$p.log 2>&1; done
timeout 600 $B --config c5 > gpurun_out/co5_c5_auto.log 2>&1
for c in c2 c3; do
CMD="python bench.py --config $c --coarse 32 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 600 $CMD > gpurun_out/co5_plain_$c.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 6000 -c 2500 --csv \
  --log-file gpurun_out/co5_launches_$c.csv $CMD > gpurun_out/co5_ncu_$c.log 2>&1
done
