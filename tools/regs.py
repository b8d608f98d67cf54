"""Registers / spills per kernel from the ptxas -v log (dev helper)."""
import re
import subprocess
import sys

log = open(sys.argv[1] if len(sys.argv) > 1 else "paper_1810_02612_b200/_lib/ptxas_kernels.log").read()
pat = sys.argv[2] if len(sys.argv) > 2 else ""
cur, sp = None, ""
for line in log.splitlines():
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip().split("(")[0]
        sp = ""
    if "spill stores" in line and " 0 bytes spill stores" not in line:
        sp = sp or line.strip()
    m = re.search(r"Used (\d+) registers", line)
    if m and cur and pat in cur:
        print(m.group(1), cur[:100], sp)
