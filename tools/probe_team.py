"""Developer probe: team block sweep step timing (PHI_TRACE=1 build), ILUT
(unit op 1) and level-1 Gauss-Seidel: phase A, phase B per step, CTA 0."""
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
a = t[5:-5]
print("ILUT(U) step median", np.median(np.diff(a[:, 0])), "phase A", np.median(a[:, 1] - a[:, 0]),
      "phase B", np.median(a[:, 2] - a[:, 1]))
