"""One line per bench JSON log: value, applies/v, K1 roofline fraction and share, non-K1 ms/iteration."""
import json
import sys

for path in sys.argv[1:]:
    lines = [x for x in open(path) if x.startswith("{")]
    if not lines:
        print(path, "NO JSON:", open(path).read()[-600:])
        continue
    d = json.loads(lines[-1])
    r, c = d["roofline"], d["config"]
    it = r["launches"] / d["steps"]
    print(f"{c['workload']}: {d['value']:.1f} v/s  applies/v {c['applies_per_v']:.1f}  K1 frac {r['frac']:.3f}  "
          f"share {r['k1_share_of_step']:.3f}  ms/step {d['ms_per_step']:.1f}  iters {it:.0f}  "
          f"non-K1 ms/iter {d['ms_per_step'] * (1 - r['k1_share_of_step']) / it:.3f}")
