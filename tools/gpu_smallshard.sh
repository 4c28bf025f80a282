#!/bin/bash
# per-rank batch size of small shards: rank 0 of an N-way split of c5 alone on one GPU, over opts.batch
cd $GRAFT_REPO_ROOT
B="python bench.py --no-cpu-baseline --no-e2e --steps 2 --warmup 3 --config c5"
for spec in "8 0" "8 192" "8 256" "8 384" "8 512" "4 0" "4 384" "4 512" "4 768" "1 768" "1 1024" "1 448"; do
  set -- $spec
  timeout 300 $B $( [ $1 -gt 1 ] && echo --emulate-rank 0/$1 ) --batch $2 > gpurun_out/ss_$1_$2.log 2>&1
  python - $1 $2 <<'PY'
import json, sys
n, b = sys.argv[1:3]
for l in open(f"gpurun_out/ss_{n}_{b}.log"):
    if l.startswith("{"):
        d = json.loads(l)
        print(f"N={n} batch={b or 'auto'} -> b={d['config']['batch']} ms/step {d['ms_per_step']:.1f} applies/v {d['config']['applies_per_v']:.1f} K1 frac {d['roofline']['frac']:.3f}")
PY
done
