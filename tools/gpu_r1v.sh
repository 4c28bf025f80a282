#!/bin/bash
cd "$(dirname "$0")/.."
for s in 16 32 64; do
  timeout 900 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --config c5 --recycle $s > gpurun_out/ag_c5_r$s.log 2>&1
done
timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --config c4 --recycle 32 > gpurun_out/ag_c4_r32.log 2>&1
