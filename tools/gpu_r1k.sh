#!/bin/bash
cd "$(dirname "$0")/.."
timeout 900 python bench.py --config c5 --steps 1 --warmup 1 --cpu-seconds 60 > gpurun_out/t_bench_c5.log 2>&1
C=c5
CMD="python bench.py --config $C --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 900 $CMD > gpurun_out/t_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k1_dgemm -s 200 -c 2 \
    -o gpurun_out/t_k1full_$C $CMD > gpurun_out/t_ncu2.log 2>&1
echo "full rc=$?" >> gpurun_out/t_plain.log
