#!/bin/bash
cd "$(dirname "$0")/.."
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/y_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/y_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/y_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/y_smoke.log
timeout 900 python bench.py > gpurun_out/y_bench_default.log 2>&1; echo "rc=$?" >> gpurun_out/y_bench_default.log
B="python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e"
for c in c1 c3 c4; do timeout 400 $B --config $c > gpurun_out/y_bench_$c.log 2>&1; done
