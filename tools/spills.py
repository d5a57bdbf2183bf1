"""Per-function stack/spill summary of the last engine build (ptxas -v)."""
import re
import sys

log = open("paper_2107_05337_b200/_lib/build.log").read().splitlines()
want = sys.argv[1] if len(sys.argv) > 1 else "ILi3E"
seen = set()
for k, line in enumerate(log):
    m = re.search(r"Function properties for (\S+)", line)
    if not m:
        continue
    name = m.group(1)
    short = re.sub(r"_ZN\d+_INTERNAL_\w+?3phi47_GLOBAL__N__\w+?_cu_[0-9a-f]+", "", name)
    short = re.sub(r"_ZN3phi47_GLOBAL__N__\w+?_cu_[0-9a-f]+", "", short)[:70]
    info = log[k + 1].strip()
    key = (short, info)
    if key in seen or (want not in name and "ILb" not in name and "gs_sweep" not in name):
        continue
    seen.add(key)
    print(f"{short:72s} {info}")
