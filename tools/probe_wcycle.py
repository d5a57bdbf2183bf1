"""Developer probe: W-cycle phase accounting (PHI_TRACE=1 build): cycles per
category over one h-multigrid W-cycle (unit op 4), CTA 0."""
import ctypes as C
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2107_05337_b200 as P  # noqa: E402
from paper_2107_05337_b200 import engine as E  # noqa: E402

p, k = int(sys.argv[1]), int(sys.argv[2])
d = P.SpatialDiscretization.build(p, k)
h = P.PMultigridHierarchy(d, 1e-4)
b1 = np.random.default_rng(1).standard_normal(d.n_free_1)
h.hmg_wcycle(b1)
E.dev_tuning(8, 8, -1)
h.hmg_wcycle(b1)
buf = np.zeros(49152, np.int64)
E.lib().phi_dev_trace(buf.ctypes.data_as(C.c_void_p), buf.size)
a = buf[33000:33030]
names = {20: "resid+restrict", 21: "prolong", 22: "coarsest LU", 23: "between"}
tot = a.sum()
for c in range(24):
    if a[c]:
        print(f"{names.get(c, f'sweeps level {c}'):16s} {a[c]:9d} cyc  {100 * a[c] / tot:5.1f}%")
print(f"total            {tot:9d} cyc")
