#!/bin/bash
# coarse pipeline: ncu launch lists of the engine kernels with the two-level preconditioner (c2 / c3)
cd $GRAFT_REPO_ROOT
python paper_2312_08201_b200/build.py > gpurun_out/co6_build.log 2>&1
for c in c2 c3; do
CMD="python bench.py --config $c --coarse 32 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 600 $CMD > gpurun_out/co6_plain_$c.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^(k_|k1_|cutlass|gemm|Kernel|sm)" \
  -s 2000 -c 2500 --csv --log-file gpurun_out/co6_launches_$c.csv $CMD > gpurun_out/co6_ncu_$c.log 2>&1
done
