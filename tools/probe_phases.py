"""Developer probe: phase stamps (pstamp ids) inside the V-cycle, for the
standalone V-cycle kernel and for the fused solve (wave) kernel."""
import ctypes as C
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2107_05337_b200 as P  # noqa: E402
from paper_2107_05337_b200 import engine as E  # noqa: E402

BASE = 40000


def stamps():
    buf = np.zeros(49152, np.int64)
    E.lib().phi_dev_trace(buf.ctypes.data_as(C.c_void_p), buf.size)
    n = min(int(buf[BASE]), 4000)
    ids = buf[BASE + 1: BASE + 1 + 2 * n: 2]
    clk = buf[BASE + 2: BASE + 2 + 2 * n: 2]
    return list(zip(ids.tolist(), clk.tolist()))


def show(tag, st):
    out = []
    for (i0, c0), (i1, c1) in zip(st, st[1:]):
        out.append(f"{i0}->{i1}:{(c1 - c0) / 1e3:.0f}k")
    print(tag, " ".join(out[:40]), flush=True)


d = P.SpatialDiscretization.build(3, 6)
h = P.PMultigridHierarchy(d, 1e-4, exact=len(sys.argv) > 1 and sys.argv[1] == "exact")
b = np.random.default_rng(0).standard_normal(d.n_free)
h.vcycle(b, np.zeros(d.n_free))
E.dev_tuning(8, 8, -1)
h.vcycle(b, np.zeros(d.n_free))
show("vcycle_kernel", stamps())
E.dev_tuning(8, 8, -1)
h.solve(b, None, fixed_cycles=1)
show("wave_kernel  ", stamps())

import time
E.dev_tuning(8, 8, 0)
x0 = np.zeros(d.n_free)
for reps in (1, 20):
    t = time.perf_counter()
    for _ in range(reps):
        h.vcycle(b, x0)
    print(f"vcycle wall {1e3 * (time.perf_counter() - t) / reps:.3f} ms/call (reps {reps})", flush=True)
