"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[start]
ix = {h: i for i, h in enumerate(hdr)}
agg = defaultdict(lambda: [0, 0.0])
for r in rows[start + 1:]:
    if len(r) < len(hdr):
        continue
    try:
        v = float(r[ix["Metric Value"]].replace(",", ""))
    except ValueError:
        continue
    name = r[ix["Kernel Name"]].split("(")[0][:70]
    agg[name][0] += 1
    agg[name][1] += v
tot = sum(t for _, t in agg.values())
print(f"{'launches':>8} {'total ms':>10} {'share':>7}  kernel")
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{c:8d} {t / 1e6:10.3f} {100 * t / tot:6.1f}%  {k}")
