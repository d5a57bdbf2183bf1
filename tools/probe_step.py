"""Developer probe: one single-RHS Phi step (the coarse march's unit of work),
wall time per step and (PHI_TRACE=1 build) phase stamps and W-cycle accounting
of CTA 0 -- cluster mode unless PHI_CLUSTER=1."""
import ctypes as C
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2107_05337_b200 as P  # noqa: E402
from paper_2107_05337_b200 import engine as E  # noqa: E402

p, k, dt = int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3])
d = P.SpatialDiscretization.build(p, k)
st = P.ThetaStepper(d, 1.0, dt, 1.0)
u = np.random.default_rng(0).uniform(-1, 1, d.n_free)
x = st.step(u)
t0 = time.perf_counter()
for _ in range(20):
    st.step(u, guess=x)
print(f"step wall {1e3 * (time.perf_counter() - t0) / 20:.3f} ms (guess = previous result)", flush=True)
u2 = np.random.default_rng(1).uniform(-1, 1, d.n_free)
t0 = time.perf_counter()
for _ in range(5):
    st.step(u2)
print(f"step wall {1e3 * (time.perf_counter() - t0) / 5:.3f} ms (zero guess)", flush=True)
if len(sys.argv) > 4:
    mask = int(sys.argv[5]) if len(sys.argv) > 5 else 0  # developer mask (c_tune.xmask)
    E.dev_tuning(-mask if mask else 8, 8, -1)
    st.step(u2)
    buf = np.zeros(49152, np.int64)
    E.lib().phi_dev_trace(buf.ctypes.data_as(C.c_void_p), buf.size)
    n = min(int(buf[40000]), 4000)
    ids = buf[40001:40001 + 2 * n:2]
    clk = buf[40002:40002 + 2 * n:2]
    from collections import defaultdict
    acc = defaultdict(int)
    for (i0, c0), (i1, c1) in zip(zip(ids, clk), zip(ids[1:], clk[1:])):
        acc[f"{i0}->{i1}"] += c1 - c0
    print("phase stamps (cycles):", dict(sorted(acc.items(), key=lambda kv: -kv[1])[:12]))
    a = buf[33000:33030]
    print("wcycle accounting:", {c: int(a[c]) for c in range(30) if a[c]})
