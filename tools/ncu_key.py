"""Key metrics of an ncu report (dev helper): time, issue, pipes, L1, stalls.

  python tools/ncu_key.py gpurun_out/x.ncu-rep [kernel-regex]
"""
import csv
import io
import subprocess
import sys

kf = ["-k", "regex:" + sys.argv[2]] if len(sys.argv) > 2 else []
txt = subprocess.run(["ncu", "-i", sys.argv[1], *kf, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(txt)))
h = r[0]
for v in r[2:]:
    d = dict(zip(h, v))
    print(d.get("Kernel Name", "?")[:60])
    for k in ["gpu__time_duration.sum", "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
              "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
              "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
              "sm__inst_executed_pipe_fmaheavy.avg.pct_of_peak_sustained_active",
              "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
              "l1tex__throughput.avg.pct_of_peak_sustained_active", "l1tex__data_pipe_lsu_wavefronts.sum",
              "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
              "sm__warps_active.avg.pct_of_peak_sustained_active", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
              "launch__registers_per_thread"]:
        if k in d:
            print(f"  {k:70s} {d[k]}")
    st = {k: d[k] for k in h if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued")}
    tot = sum(float(x or 0) for x in st.values()) or 1
    top = sorted(st.items(), key=lambda kv: -float(kv[1] or 0))[:8]
    print("  stalls:", " ".join(f"{k[33:]}={100 * float(x) / tot:.1f}%" for k, x in top))
