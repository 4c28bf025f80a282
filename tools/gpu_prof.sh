#!/bin/bash
# ncu pass on one config: launch list + full capture of the K1 GEMM.  Usage: tools/gpu_prof.sh c2 [steps]
cd "$(dirname "$0")/.."
C=${1:-c2}; S=${2:-1}
CMD="python bench.py --config $C --steps $S --warmup 1 --no-cpu-baseline --no-e2e"
timeout 600 $CMD > gpurun_out/p_plain_$C.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
    --log-file gpurun_out/p_launches_$C.csv $CMD > gpurun_out/p_ncu_launch_$C.log 2>&1
echo "launch-list rc=$?" >> gpurun_out/p_plain_$C.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k1_dgemm -s 20 -c 2 \
    -o gpurun_out/p_k1_$C $CMD > gpurun_out/p_ncu_full_$C.log 2>&1
echo "full rc=$?" >> gpurun_out/p_plain_$C.log
