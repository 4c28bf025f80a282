#!/bin/bash
# Parameter sweep of the mixed-precision engine (one gpurun call): bench lines for c5 / c4 over the
# refinement-cycle reduction mixed_eta and the restart length.  Output: gpurun_out/<prefix>_sweep.log
cd "$(dirname "$0")/.."
P=${EV_PREFIX:-sw}
OUT=gpurun_out/${P}_sweep.log
: > $OUT
run() {  # run <label> <bench args...>
  local label=$1; shift
  local line
  line=$(env $ENVS timeout 400 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e "$@" 2>>gpurun_out/${P}_err.log | tail -1)
  python - "$label" "$line" >> $OUT <<'EOF'
import json, sys
label, line = sys.argv[1], sys.argv[2]
try:
    d = json.loads(line); c = d["config"]; r = d.get("roofline", {})
    print(f"{label:40s} {d['value']:9.1f} v/s  applies/v {c.get('applies_per_v', 0):6.1f} "
          f"(exact {c.get('exact_applies_per_v', 0):5.2f})  K1 frac {r.get('frac', 0):.3f} share {r.get('k1_share_of_step', 0):.3f}"
          f"  sm {d.get('clocks', {}).get('sm_mhz')}")
except Exception as e:
    print(f"{label:40s} FAILED {e!r} {line[:200]}")
EOF
}
for spec in "$@"; do
  # spec: label|ENV=VAL ...|bench args
  label=${spec%%|*}; rest=${spec#*|}
  ENVS=${rest%%|*}; args=${rest#*|}
  run "$label" $args
done
