#!/bin/bash
# VERIFY GEMM tile configuration at the final batch size (c5 b = 1024): 0 = 64x32x16 3 stages (default), 1 = 64x64, 2 = 64x32x16 2 stages
cd $GRAFT_REPO_ROOT
B="python bench.py --no-cpu-baseline --no-e2e --steps 3 --warmup 3"
for v in 0 1 2; do LYAP_VER_CFG=$v timeout 300 $B --config c5 > gpurun_out/ver_c5_$v.log 2>&1; echo "cfg $v: $(python tools/bench_summary.py gpurun_out/ver_c5_$v.log)"; done
for v in 0 1; do LYAP_VER_CFG=$v timeout 300 $B --config c4 > gpurun_out/ver_c4_$v.log 2>&1; echo "cfg $v: $(python tools/bench_summary.py gpurun_out/ver_c4_$v.log)"; done
