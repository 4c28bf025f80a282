#!/bin/bash
cd "$(dirname "$0")/.."
B="python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e"
timeout 300 $B --config c2 --batch 2048 > gpurun_out/j_c2_b2048.log 2>&1
LYAP_GROUPS=1 timeout 300 $B --config c2 --batch 1024 > gpurun_out/j_c2_b1024_g1.log 2>&1
timeout 300 $B --config c3 --batch 2048 > gpurun_out/j_c3_b2048.log 2>&1
timeout 400 $B --config c4 --batch 2048 > gpurun_out/j_c4_b2048.log 2>&1
B5="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --config c5"
timeout 600 $B5 --batch 592 > gpurun_out/j_c5_b592.log 2>&1
LYAP_GROUPS=1 timeout 600 $B5 --batch 296 > gpurun_out/j_c5_b296_g1.log 2>&1
