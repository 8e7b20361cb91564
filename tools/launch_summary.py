"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list by kernel."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = defaultdict(lambda: [0, 0.0])
order = []
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            k = d["Kernel Name"].replace("void unnamed>::", "").split("(")[0]
            v = float(d["Metric Value"].replace(",", ""))
            if k not in agg:
                order.append(k)
            agg[k][0] += 1
            agg[k][1] += v
tot = sum(v for _, v in agg.values())
print(f"{'launches':>8} {'total us':>10} {'share':>6} {'avg us':>9}  kernel")
for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{c:8d} {v / 1e3:10.1f} {100 * v / tot:5.1f}% {v / c / 1e3:9.1f}  {k}")
