"""Developer probe: per-block stamps of the block sweeps (PHI_TRACE=1 build).
Solver warp: start, unit ready, loads issued, old sums ready, block done;
worker: progress ready, unit ready, hand-off -- cycles, CTA 0."""
import ctypes as C
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2107_05337_b200 as P  # noqa: E402
from paper_2107_05337_b200 import engine as E  # noqa: E402

BASE = 24000
p, k = int(sys.argv[1]), int(sys.argv[2])
d = P.SpatialDiscretization.build(p, k)
h = P.PMultigridHierarchy(d, 1e-4)
b = np.random.default_rng(0).standard_normal(d.n_free)
b1 = np.random.default_rng(1).standard_normal(d.n_free_1)


def trace(nb):
    buf = np.zeros(49152, np.int64)
    E.lib().phi_dev_trace(buf.ctypes.data_as(C.c_void_p), buf.size)
    t = buf[BASE:BASE + 8 * nb].reshape(nb, 8)
    return t


for name, f, n in [("ilut(U)", lambda: h.ilut_apply(b), d.n_free), ("gs0", lambda: h.gauss_seidel_sweep(0, b1, b1), d.n_free_1)]:
    f()
    E.dev_tuning(8, 8, -1)
    f()
    nb = (n + 31) // 32
    t = trace(nb)
    t0 = t[0, 0]
    per = np.diff(t[:, 3])
    print(f"{name}: nb {nb}, total {t[-1, 3] - t0} cyc, per block median {np.median(per):.0f} mean {per.mean():.0f}")
    seg = {"cntwait": t[:, 1] - t[:, 0], "pre+handwait": t[:, 2] - t[:, 1], "chain": t[:, 3] - t[:, 2], " fresh->t": t[:, 7] - t[:, 2], " t->done": t[:, 3] - t[:, 7],
           "handoff(next start - done)": np.r_[t[1:, 2] - t[:-1, 3], 0],
           "wk_mbar_done->prog": t[:, 5] - t[:, 4], "wk_prog->cnt": t[:, 6] - t[:, 5],
           "wk_cnt_vs_solver_cntwait": t[:, 6] - t[:, 0]}
    for kname, v in seg.items():
        print(f"   {kname:24s} median {np.median(v):8.0f}  mean {v.mean():8.0f}  max {v.max():8.0f}")
    print("   first blocks:", (t[:6] - t0).tolist())
