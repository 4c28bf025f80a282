#!/bin/bash
cd "$(dirname "$0")/.."
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/ad_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ad_pytest.log
B="python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e"
for c in c1 c2 c3 c4; do timeout 400 $B --config $c > gpurun_out/ad_bench_$c.log 2>&1; done
C=c2
CMD="python bench.py --config $C --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 600 $CMD > gpurun_out/ad_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed \
   --clock-control none -k regex:"^(k_|k1_)" -s 3000 -c 1400 --csv --log-file gpurun_out/ad_kern_$C.csv $CMD > gpurun_out/ad_ncu1.log 2>&1
