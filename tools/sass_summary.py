"""Per-kernel SASS mnemonic summary of the engine library (cuobjdump -sass):
instruction count and the counts of the mnemonics that show what a kernel uses
-- UBLKCP (cp.async.bulk, the TMA bulk-copy engine), SYNCS (mbarrier),
UCGABAR_ARV / UCGABAR_WAIT (cluster barriers), QSPC (address-space queries
around the distributed-shared-memory accesses, which are generic LD/ST; the
peer addresses come from SR_CgaCtaId arithmetic), DFMA/DADD/DMUL (fp64),
LDS/STS, LDG/STG, SHFL, BAR, ATOMS/REDS (shared-memory hand-offs), local-memory
spills (LDL/STL).

    python tools/sass_summary.py [lib.so] > profiles/r02/r02g_sass_summary.txt
"""
from __future__ import annotations

import collections
import re
import subprocess
import sys

LIB = sys.argv[1] if len(sys.argv) > 1 else "paper_2107_05337_b200/_lib/libphi_engine.so"
KEYS = ["UBLKCP", "SYNCS", "UCGABAR_ARV", "UCGABAR_WAIT", "QSPC", "DFMA", "DADD", "DMUL", "MUFU", "LDS", "STS", "LDG", "STG", "LD", "ST",
        "SHFL", "BAR", "ATOMS", "REDS", "ATOMG", "REDG", "LDL", "STL", "CCTL", "FENCE", "MEMBAR", "NANOSLEEP"]


def demangle(names):
    out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.split("\n")
    return dict(zip(names, out))


def main() -> None:
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
    kernels: dict[str, collections.Counter] = {}
    cur = None
    ins = re.compile(r"^\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\d+\s+)?([A-Z0-9_]+)")
    for line in sass.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            cur = kernels.setdefault(m.group(1), collections.Counter())
            continue
        if cur is None:
            continue
        m = ins.match(line)
        if m:
            cur[m.group(1)] += 1
            cur["_total"] += 1
    names = demangle(list(kernels))
    print(f"# {LIB}: {len(kernels)} kernels, arch sm_100a; counts of static SASS instructions")
    print("# kernel | total | " + " ".join(KEYS))
    for k, c in sorted(kernels.items(), key=lambda kv: -kv[1]["_total"]):
        short = names[k].replace("(anonymous namespace)::", "")
        short = re.sub(r"^void ", "", re.sub(r"\(.*", "", short))
        print(f"{short} | {c['_total']} | " + " ".join(f"{key}={c[key]}" for key in KEYS if c[key]))


if __name__ == "__main__":
    main()
