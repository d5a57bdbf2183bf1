"""Summarise ptxas register / spill lines of the last engine build per kernel."""
import re
import sys

log = open("paper_2107_05337_b200/_lib/build.log").read().splitlines()
want = sys.argv[1] if len(sys.argv) > 1 else "ILi3E"
cur = None
for line in log:
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = m.group(1)
        continue
    if cur and want in cur and ("registers" in line or "spill" in line):
        name = re.sub(r"_ZN3phi\w+?_GLOBAL__N__\w+?_phi_kernels_cu_\w+?(\d+)", r"\1", cur)[:60]
        print(f"{name:60s} {line.split(':', 1)[1].strip()}")
