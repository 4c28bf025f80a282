#!/bin/bash
# launch order A/B at the final batch size (c5 b = 1024, c4 b = 2000)
cd $GRAFT_REPO_ROOT
B="python bench.py --no-cpu-baseline --no-e2e --steps 3 --warmup 3"
for o in 1 0 1 0; do LYAP_MP_ORDER=$o timeout 300 $B --config c5 > gpurun_out/ord2_c5_o${o}.log 2>&1; echo "order $o: $(python tools/bench_summary.py gpurun_out/ord2_c5_o${o}.log)"; done
for o in 1 0; do LYAP_MP_ORDER=$o timeout 300 $B --config c4 > gpurun_out/ord2_c4_o${o}.log 2>&1; echo "order $o: $(python tools/bench_summary.py gpurun_out/ord2_c4_o${o}.log)"; done
