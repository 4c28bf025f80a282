#!/bin/bash
# c2 batch / restart-length sweep after the chain-kernel changes
B="python bench.py --no-cpu-baseline --no-e2e --config c2 --steps 3 --warmup 3"
for b in 512 768 1024 1536 2048; do timeout 300 $B --batch $b > gpurun_out/sw_b$b.json 2>&1; done
for m in 96 128 200; do timeout 300 $B --max-dim $m > gpurun_out/sw_m$m.json 2>&1; done
B4="python bench.py --no-cpu-baseline --no-e2e --config c4 --steps 2 --warmup 3"
for b in 1024 2048; do timeout 400 $B4 --batch $b > gpurun_out/sw4_b$b.json 2>&1; done
