"""Per-kernel share of device time from an ncu launch list (gpu__time_duration.sum)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, mi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = collections.defaultdict(lambda: [0, 0.0])
mult = {"usecond": 1e-3, "us": 1e-3, "nsecond": 1e-6, "ns": 1e-6, "msecond": 1.0, "ms": 1.0}
for r in rows[hi + 1:]:
    if len(r) <= mi:
        continue
    v = float(r[mi].replace(",", "")) * mult.get(r[ui], 1.0)
    name = r[ki].split("(")[0][:60]
    agg[name][0] += 1
    agg[name][1] += v
tot = sum(v[1] for v in agg.values())
for k, (c, ms) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:60s} n={c:4d} total={ms:9.3f} ms share={ms / tot * 100:5.1f}%")
