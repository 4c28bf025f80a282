#!/bin/bash
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests -m gpu -x -q -k "recycle" > gpurun_out/x_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/x_pytest.log
B="python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e"
for s in 32 64; do timeout 400 $B --config c2 --recycle $s > gpurun_out/x_c2_r$s.log 2>&1; done
timeout 600 $B --config c4 --recycle 64 > gpurun_out/x_c4_r64.log 2>&1
for s in 32 64 128; do timeout 900 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --config c5 --recycle $s > gpurun_out/x_c5_r$s.log 2>&1; done
