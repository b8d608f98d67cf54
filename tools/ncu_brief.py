"""Key counters + stall mix of an ncu report (dev helper)."""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = list(csv.reader(io.StringIO(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                                                 text=True).stdout)))
h = raw[0]
for row in raw[2:]:
    d = dict(zip(h, row))
    print(d["Kernel Name"].split("(")[0][:100])
    for k in ["gpu__time_duration.sum", "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
              "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes_read.sum", "dram__bytes_write.sum",
              "l1tex__throughput.avg.pct_of_peak_sustained_active", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
              "l1tex__m_xbar2l1tex_read_sectors_mem_lg_op_ld.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
              "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread"]:
        print(f"  {k:60s} {d.get(k)}")
src = list(csv.reader(io.StringIO(subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                                                 capture_output=True, text=True).stdout)))
hs = src[1]
c = collections.Counter()
for r in src[2:]:
    d = dict(zip(hs, r))
    for k in hs:
        if k.startswith("stall_") and "Not Issued" not in k:
            try:
                c[k[6:]] += float(d.get(k, 0) or 0)
            except (ValueError, TypeError):
                pass
t = sum(c.values())
print("  stalls: " + " ".join(f"{k}={100 * v / t:.1f}%" for k, v in c.most_common(9)))
