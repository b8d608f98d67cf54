"""Write the committed evidence for one GPU pass: profiles/<name>_ncu_summary.md
(launch list shares + key counters + SASS mix of both labeling kernels),
<name>_bench.json, <name>_bench_ref.json, <name>_launches.csv, and update
profiles/traffic.json (dram bytes per launch, read by bench.py).

  python tools/make_profile_summary.py gpurun_out/r02 profiles/round1
"""
import csv
import io
import json
import os
import shutil
import subprocess
import sys

src, dst = sys.argv[1], sys.argv[2]
here = os.path.dirname(os.path.abspath(__file__))
lines = []


def run(*cmd):
    return subprocess.run(list(cmd), capture_output=True, text=True).stdout


lines.append(f"# {os.path.basename(dst)}: ncu evidence (`tools/gpu_full.sh`, one B200, `--clock-control none`)\n")
lines.append("## Launch list of `python bench.py --quick --steps 3 --warmup 3 --no-cpu-baseline`")
lines.append("(gpu__time_duration.sum; cold-cache and serialised, so compare shares, not absolutes)\n```")
lines.append(run("python", os.path.join(here, "ncu_launches.py"), src + "_launches.csv").rstrip())
lines.append("```")
traffic_path = os.path.join(os.path.dirname(dst), "traffic.json")
traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
lim_path = os.path.join(os.path.dirname(dst), "limiters.json")
limiters = json.load(open(lim_path)) if os.path.exists(lim_path) else {}
TITLES = {"batch": "config 4, multi-frame labeling kernel", "stream": "config 3, single-frame labeling kernel",
          "cfg5batch": "config 5 shard (1M rows, 1024^2, 64 props), 64-frame labeling kernel",
          "cfg5stream": "config 5 shard (1M rows, 1024^2, 64 props), single-frame labeling kernel",
          "cfg5tc": "config 5 shard, 64 frames: the tcgen05 kind::i8 formulation (LTLG_TC=1; measured, dropped)"}
for kind in ("batch", "stream", "cfg5batch", "cfg5stream", "cfg5tc"):
    rep = f"{src}_{kind}.ncu-rep"
    if not os.path.exists(rep):
        continue
    lines.append(f"\n## `ncu --set full`: {TITLES[kind]}\n```")
    lines.append(run("python", os.path.join(here, "ncu_brief.py"), rep).rstrip())
    raw = list(csv.reader(io.StringIO(run("ncu", "-i", rep, "--page", "raw", "--csv"))))
    rows = [dict(zip(raw[0], r)) for r in raw[2:]]
    d = next((r for r in rows if "label_" in r.get("Kernel Name", "")), rows[0])  # the labelling kernel of the capture
    u = dict(zip(raw[0], raw[1]))
    for k in ["sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
              "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
              "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
              "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
              "smsp__thread_inst_executed_per_inst_executed.ratio"]:
        lines.append(f"  {k:60s} {d.get(k)}")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    tb = sum(float(d[k]) * scale.get(u[k], 1) for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
    full_name = d["Kernel Name"]
    name = full_name.split("(")[0].split("<")[0].replace("void ", "").split("::")[-1]
    if "unsigned long" in full_name.split("(")[0]:  # the 64-prop instantiations (template arguments)
        name += "<u64,2>" if "label_wm" in name else "<64>"
    traffic[name] = tb

    def pct(k):
        try:
            return round(float(d[k]), 1)
        except (KeyError, ValueError):
            return None
    # what binds the kernel, from the same capture (bench.py reports it next to the roofline)
    def cnt(k):
        try:
            return float(d[k])
        except (KeyError, ValueError):
            return None
    limiters[name] = {
        "warp_insts": cnt("smsp__inst_executed.sum"),
        "l1_data_pipe_wavefronts": (cnt("SM_A.TriageCompute.l1tex__data_pipe_lsu_wavefronts.avg")
                                    or cnt("l1tex__data_pipe_lsu_wavefronts.avg") or 0) * 148 or None,
        "kernel_ms_under_ncu": (cnt("gpu__time_duration.sum") or 0) * {"msecond": 1.0, "ms": 1.0, "usecond": 1e-3, "us": 1e-3, "ns": 1e-6,
                                                                       "nsecond": 1e-6}.get(u.get("gpu__time_duration.sum"), 1.0),
        "l1tex_data_pipe_pct": pct("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed"),
        "issue_active_pct": pct("smsp__issue_active.avg.pct_of_peak_sustained_active"),
        "dram_pct": pct("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
        "alu_pipe_pct": pct("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
        "warps_active_pct": pct("sm__warps_active.avg.pct_of_peak_sustained_active"),
        "source": os.path.basename(dst) + "_ncu_summary.md",
    }
    lines.append(f"  dram read+write bytes per launch (traffic)                   {tb:.4g}")
    lines.append(run("python", os.path.join(here, "ncu_sass.py"), rep, "12").rstrip())
    lines.append("```")
open(dst + "_ncu_summary.md", "w").write("\n".join(lines) + "\n")
json.dump(traffic, open(traffic_path, "w"), indent=1)
json.dump(limiters, open(lim_path, "w"), indent=1)
for suffix in ("_bench.json", "_bench_ref.json", "_launches.csv"):
    if os.path.exists(src + suffix):
        shutil.copy(src + suffix, dst + suffix)
print("wrote", dst + "_ncu_summary.md", traffic)
