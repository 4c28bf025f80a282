#!/bin/bash
# c5: restart length and recycle-space size around the automatic defaults (384, s = 32)
B="python bench.py --no-cpu-baseline --no-e2e --config c5 --steps 1 --warmup 3"
for m in 320 448; do timeout 400 $B --max-dim $m > gpurun_out/c5_m$m.json 2>&1; done
for s in 24 48; do timeout 400 $B --recycle $s > gpurun_out/c5_s$s.json 2>&1; done
