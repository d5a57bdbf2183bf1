"""Developer probe (PHI_TRACE=1 build): phase stamps of one single-CTA Phi step
whose guess already solves the system (zero p-MG cycles: the cost every MGRIT
solve pays before / without its V-cycles).  PHI_CLUSTER=0 python tools/probe_point.py p k dt"""
import ctypes as C
import os
import sys
from collections import defaultdict

import numpy as np

os.environ.setdefault("PHI_TRACE", "1")
os.environ.setdefault("PHI_CLUSTER", "0")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2107_05337_b200 as P  # noqa: E402
from paper_2107_05337_b200 import engine as E  # noqa: E402

p, k, dt = int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3])
E.lib().phi_set_device(0)
d = P.SpatialDiscretization.build(p, k)
st = P.ThetaStepper(d, 1.0, dt, 1.0)
u = np.random.default_rng(0).uniform(-1, 1, d.n_free)
x = st.step(u)
x = st.step(u, guess=x)
E.dev_tuning(8, 8, -1)
x2 = st.step(u, guess=x)
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
print(f"p={p} k={k}: single-CTA Phi with a solved guess: {(clk[-1] - clk[0]) / 1e6:.3f} Mcycles, stamps {n}")
for key, v in sorted(acc.items(), key=lambda kv: -kv[1])[:10]:
    print(f"  {key:8s} {v / 1e3:9.1f} kcyc  x{cnt[key]}")
