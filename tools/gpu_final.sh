#!/bin/bash
# round-end evidence for the final build: tests, smoke, default bench, per-kernel launch list, K1 full capture (c2)
cd "$(dirname "$0")/.."
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/f_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/f_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/f_smoke.log
timeout 900 python bench.py > gpurun_out/f_bench_default.log 2>&1; echo "rc=$?" >> gpurun_out/f_bench_default.log
B="python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e"
for c in c1 c3 c4; do timeout 400 $B --config $c > gpurun_out/f_bench_$c.log 2>&1; done
timeout 900 python bench.py --config c5 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/f_bench_c5.log 2>&1
C=c2
CMD="python bench.py --config $C --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 600 $CMD > gpurun_out/f_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed \
   --clock-control none -k regex:"^(k_|k1_)" -s 3000 -c 1400 --csv --log-file gpurun_out/f_kern_$C.csv $CMD > gpurun_out/f_ncu1.log 2>&1
echo "launch rc=$?" >> gpurun_out/f_plain.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k1_dgemm -s 40 -c 2 \
    -o gpurun_out/f_k1full_$C $CMD > gpurun_out/f_ncu2.log 2>&1
echo "full rc=$?" >> gpurun_out/f_plain.log
