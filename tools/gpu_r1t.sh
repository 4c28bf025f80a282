#!/bin/bash
cd "$(dirname "$0")/.."
B="python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e"
for md in 224; do
  for c in c2 c4; do timeout 400 $B --config $c --max-dim $md > gpurun_out/ae_${md}_$c.log 2>&1; done
  timeout 900 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --config c5 --max-dim $md > gpurun_out/ae_${md}_c5.log 2>&1
done
timeout 900 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --config c5 > gpurun_out/ae_160_c5.log 2>&1
