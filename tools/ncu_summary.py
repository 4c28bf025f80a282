"""Summarise an ncu --csv launch list: time share, DRAM bytes and bandwidth per kernel name."""
import collections
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h, data = rows[hi], rows[hi + 1:]
    ki, mi, vi, ui, ii = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
    per = collections.defaultdict(dict)
    names = {}
    for r in data:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        unit = r[ui]
        if unit in ("Kbyte",):
            v *= 1e3
        elif unit in ("Mbyte",):
            v *= 1e6
        elif unit in ("Gbyte",):
            v *= 1e9
        elif unit == "us":
            v *= 1e3
        elif unit == "ms":
            v *= 1e6
        per[r[ii]][r[mi]] = v
        names[r[ii]] = r[ki].split("(")[0].replace("void ", "").replace("lyap::", "")
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
    for i, m in per.items():
        a = agg[names[i]]
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0.0)
        a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
        a[3] += m.get("sm__throughput.avg.pct_of_peak_sustained_elapsed", 0.0)
    T = sum(a[1] for a in agg.values())
    print(f"{'kernel':38s} {'n':>5s} {'ms':>9s} {'share':>6s} {'GB/s':>8s} {'sm%':>5s}")
    for k, a in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k[:38]:38s} {a[0]:5d} {a[1] / 1e6:9.2f} {100 * a[1] / T:5.1f}% {a[2] / max(a[1], 1):8.1f} {a[3] / a[0]:5.1f}")
    print(f"total {T / 1e6:.2f} ms")


if __name__ == "__main__":
    main(sys.argv[1])
