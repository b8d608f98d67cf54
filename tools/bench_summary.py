"""Print the key numbers of a bench.py JSON line (dev helper)."""
import json
import sys

d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
r = d.get("roofline") or {}
lat = d.get("latency") or {}
print(f"value={d['value']:.4g} ms/step={d['ms_per_step']:.3f} label_kernel_ms={r.get('kernel_ms', 0):.3f} "
      f"summary_ms={r.get('summary_kernel_ms', 0):.4f} frac={r.get('frac', 0):.3f}")
if lat:
    print(f"cfg3 p50={lat['p50_ms']:.4f}ms kernel_p50={lat['kernel_p50_ms']:.4f}ms frac={lat['roofline']['frac']:.3f}")
if d.get("e2e"):
    print(f"e2e={d['e2e']['value']:.4g}")
if d.get("cpu_baseline"):
    print(f"cpu={d['cpu_baseline']['value']:.4g} ({d['cpu_baseline']['kind']}, {d['cpu_baseline']['cores']} cores)")
print("clocks", d.get("clocks"))
