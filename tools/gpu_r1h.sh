#!/bin/bash
# official-style bench line for c2 + ncu evidence (launch list, full capture of K1)
cd "$(dirname "$0")/.."
timeout 600 python bench.py > gpurun_out/l_bench_default.log 2>&1
C=c2
CMD="python bench.py --config $C --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 600 $CMD > gpurun_out/l_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed \
   --clock-control none -k regex:"^(k_|k1_)" -s 3000 -c 1300 --csv --log-file gpurun_out/l_kern_$C.csv $CMD > gpurun_out/l_ncu1.log 2>&1
echo "launch rc=$?" >> gpurun_out/l_plain.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k1_dgemm -s 40 -c 3 \
    -o gpurun_out/l_k1full_$C $CMD > gpurun_out/l_ncu2.log 2>&1
echo "full rc=$?" >> gpurun_out/l_plain.log
