"""Developer probe: per-block phase timing of the warp triangular solve
(trace stamps in tri_solve_warp) for one ILUT application (L then U)."""
import ctypes as C
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2107_05337_b200 as P  # noqa: E402
from paper_2107_05337_b200 import engine as E  # noqa: E402

BASE = 24000
d = P.SpatialDiscretization.build(3, 6)
h = P.PMultigridHierarchy(d, 1e-4, exact=len(sys.argv) > 1 and sys.argv[1] == "exact")
r = np.random.default_rng(0).standard_normal(d.n_free)
h.ilut_apply(r)
for kind in ("unit", "solve"):
    E.dev_tuning(8, 8, -1)
    if kind == "unit":
        h.ilut_apply(r)
    else:
        h.solve(r, None, fixed_cycles=1)
    buf = np.zeros(49152, np.int64)
    E.lib().phi_dev_trace(buf.ctypes.data_as(C.c_void_p), buf.size)
    t = buf[BASE:BASE + 8 * 1024].reshape(1024, 8).astype(np.float64)
    nb = int((t[:, 0] > 0).sum())
    t = t[:nb]
    prep = t[:, 1] - t[:, 0]
    wait = t[:, 2] - t[:, 1]
    chain = t[:, 3] - t[:, 2]
    period = np.diff(t[:, 2])
    walk = t[4:, 0] - t[:-4, 3]
    wk = buf[BASE + 8192:BASE + 8192 + 4096].reshape(4, 1024).astype(np.float64)
    for w in range(2):
        d = np.diff(wk[w, :nb])
        print(f"   warp {w} loop-top deltas (first 16):", d[:16].astype(int).tolist())
    print("   walk (chain end -> prep of the warp's next block)", float(np.median(walk)))
    med = lambda v: float(np.median(v))
    print(f"{kind}: blocks {nb}  prep {med(prep):.0f}  wait {med(wait):.0f}  chain {med(chain):.0f}  "
          f"period {med(period):.0f} / mean {period.mean():.0f} cycles")
