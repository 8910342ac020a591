"""Per-kernel share of an ncu launch list (gpu__time_duration.sum CSV)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[start]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
d = collections.defaultdict(list)
for r in rows[start + 1:]:
    if len(r) > vi and r[mi] == "gpu__time_duration.sum":
        d[r[ki].split("(")[0].replace("void ", "")[:64]].append(float(r[vi].replace(",", "")))
tot = sum(sum(v) for v in d.values())
for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k:64s} n={len(v):4d} mean={sum(v) / len(v) / 1e3:8.2f} us share={sum(v) / tot * 100:5.1f}%")
