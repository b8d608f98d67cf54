"""Summarise an ncu report's SASS page: instructions executed per opcode and
the hottest instructions by stall samples (dev helper).

  python tools/ncu_sass.py gpurun_out/r01_stream.ncu-rep [top] [kernel-regex]
"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
kfilter = ["-k", "regex:" + sys.argv[3]] if len(sys.argv) > 3 else []
txt = subprocess.run(["ncu", "-i", rep, *kfilter, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]


def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


tot = sum(num(d["Instructions Executed"]) for d in data)
samples = sum(num(d["Warp Stall Sampling (All Samples)"]) for d in data)
by_op = collections.Counter()
for d in data:
    op = d["Source"].split()[0] if d["Source"].split() else "?"
    if op.startswith("@"):
        op = d["Source"].split()[1]
    by_op[op.split(".")[0]] += num(d["Instructions Executed"])
print(f"warp instructions executed: {tot:.4g}   stall samples: {samples:.0f}")
for op, n in by_op.most_common(20):
    print(f"  {op:10s} {n:12.4g}  {100 * n / tot:5.1f}%")
print("hottest instructions (stall samples, executed):")
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
for d in sorted(data, key=lambda d: -num(d["Warp Stall Sampling (All Samples)"]))[:top]:
    reasons = sorted(((num(d[c]), c[6:]) for c in stall_cols), reverse=True)[:2]
    rs = ", ".join(f"{r}={int(v)}" for v, r in reasons if v)
    print(f"  {d['Address'][-5:]} {num(d['Warp Stall Sampling (All Samples)']):6.0f} "
          f"{num(d['Instructions Executed']):10.4g}  {d['Source'].strip()[:60]:60s} {rs}")
