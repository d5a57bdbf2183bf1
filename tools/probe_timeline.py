"""Developer probe: block-sweep timeline (PHI_TRACE=1 build), ILUT U solve
(unit op 1), CTA 0.  Solver: 0 start, 1 count seen, 2 hand-off done, 3 t, 4 z,
5 signalled, 6 post done; worker part 0: 8 unit ready, 9 loads issued, 10 prog
seen, 11 counted."""
import ctypes as C
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2107_05337_b200 as P  # noqa: E402
from paper_2107_05337_b200 import engine as E  # noqa: E402

p, k = int(sys.argv[1]), int(sys.argv[2])
d = P.SpatialDiscretization.build(p, k)
h = P.PMultigridHierarchy(d, 1e-4)
b = np.random.default_rng(0).standard_normal(d.n_free)
nb = (d.n_free + 31) // 32
h.ilut_apply(b)
E.dev_tuning(8, 8, -1)
h.ilut_apply(b)
buf = np.zeros(49152, np.int64)
E.lib().phi_dev_trace(buf.ctypes.data_as(C.c_void_p), buf.size)
t = buf[24000:24000 + 16 * min(nb, 512)].reshape(-1, 16)
t0 = t[40, 0]
print("blk  start  cnt   hand   t      z      sig    post | wk: unit  loads  prog  cnt")
for g in range(40, 52):
    r = t[g] - t0
    print(g, " ".join(f"{v:6d}" for v in r[:7]), "|", " ".join(f"{v:6d}" for v in r[8:12]))
per = np.diff(t[:, 5])
print("per block median", np.median(per[10:-10]))
for nm, a, bb in [("cntwait", 0, 1), ("pre (y ready)", 1, 2), ("handwait", 2, 3), ("chain", 3, 5), ("post", 5, 6),
                  ("wk unit->loads", 8, 9), ("wk loads->prog", 9, 10), ("wk prog->cnt", 10, 11)]:
    v = t[10:-10, bb] - t[10:-10, a]
    print(f"  {nm:16s} median {np.median(v):7.0f}")
