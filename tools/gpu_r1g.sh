#!/bin/bash
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/o_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/o_pytest.log
B="python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e"
for c in c1 c2 c3 c4; do timeout 400 $B --config $c > gpurun_out/o_bench_$c.log 2>&1; done
timeout 600 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --config c5 > gpurun_out/o_bench_c5.log 2>&1
