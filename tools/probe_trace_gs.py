"""Trace per-wavefront clock64 stamps of the sync-free Gauss-Seidel sweep."""
import ctypes as C
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2107_05337_b200 as P  # noqa: E402
from paper_2107_05337_b200.engine import lib  # noqa: E402

d = P.SpatialDiscretization.build(3, 6)
h = P.PMultigridHierarchy(d, 1e-4)
r1 = np.random.default_rng(1).standard_normal(d.n_free_1)
h.gauss_seidel_sweep(0, r1, r1)
lib().phi_dev_tuning(8, 8, -1)
h.gauss_seidel_sweep(0, r1, r1)
buf = np.zeros(8 * 1024 * 6, np.int64)
lib().phi_dev_trace.argtypes = [C.c_void_p, C.c_int]
lib().phi_dev_trace(buf.ctypes.data, buf.size)
g = buf[8 * 1024 * 2:8 * 1024 * 6].reshape(8, 1024, 4)
t0 = g[:, :, 0][g[:, :, 0] > 0].min()
for w in range(3):
    nz = g[w, :, 0] > 0
    a = g[w, nz, 0] - t0
    b = g[w, nz, 1] - t0
    c = g[w, nz, 2] - t0
    print(f"warp {w} items={nz.sum()} start={a[:8]}")
    print("   wait(ready-start)=", (b - a)[:10], " compute(end-ready)=", (c - b)[:10])
    print("   gaps:", np.diff(a)[:10])
allv = g[:, :, 0] > 0
print("span", (g[:, :, 2][allv] - t0).max(), "items", allv.sum())
# chain analysis: wavefront t handled by warp t % 16, item t // 16
S, R, E = {}, {}, {}
for t in range(187):
    w, k = t % 8, t // 8
    if g[w, k, 0] > 0:
        S[t], R[t], E[t] = g[w, k, 0] - t0, g[w, k, 1] - t0, g[w, k, 2] - t0
hop = [R[t] - E[t - 1] for t in range(1, 187) if t in R and t - 1 in E]
comp = [E[t] - R[t] for t in R]
late = [S[t] - E[t - 1] for t in range(1, 187) if t in S and t - 1 in E]
print("ready - prev_end: median", np.median(hop), "p90", np.percentile(hop, 90))
print("end - ready: median", np.median(comp))
print("start - prev_end (neg = started early): median", np.median(late), "p10", np.percentile(late, 10), "p90", np.percentile(late, 90))
print("per-wavefront period", (E[186] - E[0]) / 186 if 186 in E else None)
