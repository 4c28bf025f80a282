#!/bin/bash
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/u_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/u_pytest.log
B="python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e"
for c in c2 c4; do timeout 400 $B --config $c > gpurun_out/u_bench_$c.log 2>&1; done
C=c5
CMD="python bench.py --config $C --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 900 $CMD > gpurun_out/u_bench_c5.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k1_dgemm -s 200 -c 2 \
    -o gpurun_out/u_k1full_$C $CMD > gpurun_out/u_ncu2.log 2>&1
echo "full rc=$?" >> gpurun_out/u_bench_c5.log
