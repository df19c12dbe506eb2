"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
H = rows[hdr]
ki, vi, ui = H.index("Kernel Name"), H.index("Metric Value"), H.index("Metric Unit")
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[hdr + 1:]:
    name = r[ki].split("(")[0].replace("void ", "")
    name = name.replace("glod::<unnamed>::", "").replace("glod::(anonymous namespace)::", "")
    name = name[:60]
    v = float(r[vi].replace(",", ""))
    v = v / 1e3 if r[ui] == "ns" else (v * 1e3 if r[ui] == "ms" else v)
    agg[name][0] += 1
    agg[name][1] += v
tot = sum(v[1] for v in agg.values())
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
print(f"{'us/step':>10} {'share':>6} {'n':>5}  kernel")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{v[1] / steps:10.1f} {100 * v[1] / tot:5.1f}% {v[0]:5d}  {k}")
print(f"total {tot / steps:.1f} us/step over {steps} steps, {sum(v[0] for v in agg.values())} launches")
