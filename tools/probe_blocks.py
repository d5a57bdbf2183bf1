"""Developer probe (PHI_TRACE=1 build): per-block timing of the block-recurrence
sweeps and phase stamps of one single-RHS Phi step (the coarse march's unit
of work).  python tools/probe_blocks.py p k dt"""
import ctypes as C
import os
import sys
import time
from collections import defaultdict

import numpy as np

os.environ.setdefault("PHI_TRACE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2107_05337_b200 as P  # noqa: E402
from paper_2107_05337_b200 import engine as E  # noqa: E402

p, k, dt = int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3])
E.lib().phi_set_device(0)
d = P.SpatialDiscretization.build(p, k)
st = P.ThetaStepper(d, 1.0, dt, 1.0)
u = np.random.default_rng(0).uniform(-1, 1, d.n_free)
st.step(u)
t0 = time.perf_counter()
for _ in range(5):
    st.step(u)
print(f"p={p} k={k}: step wall {1e3 * (time.perf_counter() - t0) / 5:.3f} ms (zero guess)", flush=True)
E.dev_tuning(8, 8, -1)
st.step(u)
buf = np.zeros(49152, np.int64)
E.lib().phi_dev_trace(buf.ctypes.data_as(C.c_void_p), buf.size)
n = min(int(buf[40000]), 4000)
ids = buf[40001:40001 + 2 * n:2]
clk = buf[40002:40002 + 2 * n:2]
acc = defaultdict(int)
cnt = defaultdict(int)
for (i0, c0), (i1, c1) in zip(zip(ids, clk), zip(ids[1:], clk[1:])):
    acc[f"{i0}->{i1}"] += c1 - c0
    cnt[f"{i0}->{i1}"] += 1
tot = clk[-1] - clk[0] if n else 0
print(f"phase stamps: total {tot / 1e6:.2f} Mcycles")
for key, v in sorted(acc.items(), key=lambda kv: -kv[1])[:14]:
    print(f"  {key:8s} {v / 1e6:8.3f} Mcyc  x{cnt[key]}  {v / cnt[key] / 1e3:.1f} kcyc each")
a = buf[33000:33030]
print("wcycle accounting (Mcyc):", {c: round(int(a[c]) / 1e6, 3) for c in range(30) if a[c]})
# per-block trace of the last block sweep (first 512 blocks)
T = buf[24000:24000 + 16 * 512].reshape(512, 16)
ok = T[:, 5] > 0
g = np.nonzero(ok)[0]
if len(g) > 8:
    g = g[2:]
    done = T[g, 5]
    per = np.diff(done)
    print(f"blocks traced {len(g)}: per-block {np.median(per):.0f} cycles (median), p90 {np.percentile(per, 90):.0f}")
    print(f"  unit landed (1-0) {np.median(T[g, 1] - T[g, 0]):.0f}, inverse + G loads (7-1) {np.median(T[g, 7] - T[g, 1]):.0f}, "
          f"parts + inverse product (4-7) {np.median(T[g, 4] - T[g, 7]):.0f}, hand wait (2-4) {np.median(T[g, 2] - T[g, 4]):.0f}, "
          f"chain (3-2) {np.median(T[g, 3] - T[g, 2]):.0f}, store+signal (5-3) {np.median(T[g, 5] - T[g, 3]):.0f}, "
          f"bookkeeping (6-5) {np.median(T[g, 6] - T[g, 5]):.0f}")
    w = T[g, 8] > 0
    if w.any():
        gw = g[w]
        print(f"  worker0: unit wait {np.median(T[gw, 9] - T[gw, 8]):.0f}, prog wait {np.median(T[gw, 10] - T[gw, 9]):.0f}, "
              f"sum+publish {np.median(T[gw, 11] - T[gw, 10]):.0f}")
