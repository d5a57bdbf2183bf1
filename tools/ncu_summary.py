"""Summarise ncu outputs for profiles/.

  python tools/ncu_summary.py launches <launches.csv>      per-kernel share of GPU time
  python tools/ncu_summary.py full <report.ncu-rep>        key metrics of a --set full capture
  python tools/ncu_summary.py raw <raw.csv>                the same from `ncu -i .. --page raw --csv` output
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0].replace("(anonymous namespace)::", "")
        agg[name][0] += 1
        agg[name][1] += float(r[vi].replace(",", ""))
    total = sum(v[1] for v in agg.values())
    out = []
    for name, (cnt, ns) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out.append({"kernel": name, "launches": cnt, "total_ms": ns / 1e6, "avg_us": ns / cnt / 1e3,
                    "share": ns / total})
    return {"total_ms": total / 1e6, "launches": sum(v[0] for v in agg.values()), "kernels": out}


WANT = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
    "launch__block_size", "launch__shared_mem_per_block_dynamic", "smsp__inst_executed.sum",
    "lts__t_bytes.sum", "l1tex__t_bytes.sum", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
]


def full(path, raw_csv=False):
    if raw_csv:
        txt = open(path).read()
    else:
        txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = [r for r in csv.reader(io.StringIO(txt)) if len(r) > 10]
    hdr, units, data = rows[0], rows[1], rows[2:]
    res = []
    for r in data:
        d = {"kernel": r[hdr.index("Kernel Name")].split("(")[0]}
        for m in WANT:
            if m in hdr:
                d[m] = r[hdr.index(m)] + ("" if not units[hdr.index(m)] else " " + units[hdr.index(m)])
        stalls = {}
        for i, h in enumerate(hdr):
            if h.startswith("smsp__average_warp_latency_issue_stalled_") or (
                    h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued")):
                try:
                    stalls[h] = float(r[i].replace(",", ""))
                except ValueError:
                    pass
        top = sorted(stalls.items(), key=lambda kv: -kv[1])[:8]
        d["top_stalls"] = top
        res.append(d)
    return res


if __name__ == "__main__":
    kind, path = sys.argv[1], sys.argv[2]
    print(json.dumps(launches(path) if kind == "launches" else full(path, raw_csv=kind == "raw"), indent=1))
