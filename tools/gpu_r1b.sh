#!/bin/bash
# round-1 second GPU pass: full parity tests (incl. c4/c5), bench sweep, ncu on c2
cd "$(dirname "$0")/.."
timeout 1500 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/b_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/b_pytest.log
for md in 40 80 160; do
  timeout 300 python bench.py --config c2 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --max-dim $md > gpurun_out/b_bench_c2_m$md.log 2>&1; echo "rc=$?" >> gpurun_out/b_bench_c2_m$md.log
done
timeout 300 python bench.py --config c3 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/b_bench_c3.log 2>&1
timeout 600 python bench.py --config c4 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/b_bench_c4.log 2>&1
timeout 900 python bench.py --config c5 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/b_bench_c5.log 2>&1
timeout 300 python bench.py --config c2 --steps 3 --warmup 3 --cpu-seconds 15 > gpurun_out/b_bench_c2_full.log 2>&1
bash tools/gpu_prof.sh c2 1
