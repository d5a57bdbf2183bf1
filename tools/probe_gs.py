"""ncu target: single-CTA Gauss-Seidel sweeps on the finest order-1 level."""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2107_05337_b200 as P  # noqa: E402

p, k = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (3, 6)
d = P.SpatialDiscretization.build(p, k)
h = P.PMultigridHierarchy(d, 1e-4)
r1 = np.random.default_rng(1).standard_normal(d.n_free_1)
for _ in range(3):
    x = h.gauss_seidel_sweep(0, r1, r1)
print("ok", float(np.abs(x).sum()))
