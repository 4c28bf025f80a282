#!/bin/bash
# per-kernel time + DRAM bytes for the engine kernels (skip setup/warmup launches)
cd "$(dirname "$0")/.."
for C in ${CFGS:-c2 c5}; do
  CMD="python bench.py --config $C --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
  timeout 900 $CMD > gpurun_out/q_plain_$C.log 2>&1 && \
  timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed \
     --clock-control none -k regex:"^(k_|k1_)" -s 3000 -c 660 --csv --log-file gpurun_out/q_kern_$C.csv $CMD > gpurun_out/q_ncu_$C.log 2>&1
  echo "rc=$?" >> gpurun_out/q_plain_$C.log
done
