"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv):
launches, total and mean device time per kernel, and each kernel's share.

  python tools/ncu_launches.py gpurun_out/r01_launches.csv
"""
import collections
import csv
import sys

SCALE = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
rows = list(csv.reader(open(sys.argv[1])))
i = next(k for k, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[i]
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[i + 1:]:
    d = dict(zip(hdr, r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = d["Kernel Name"].split("(")[0].replace("void ", "")
    agg[name][0] += 1
    agg[name][1] += float(d["Metric Value"].replace(",", "")) * SCALE[d["Metric Unit"]]
tot = sum(t for _, t in agg.values())
print(f"{'launches':>8} {'total us':>11} {'mean us':>10} {'share':>6}  kernel")
for name, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{n:8d} {t:11.1f} {t / n:10.2f} {100 * t / tot:5.1f}%  {name}")
