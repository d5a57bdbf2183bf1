"""Developer driver: one level-0 Gauss-Seidel sweep (unit op 5) for ncu."""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2107_05337_b200 as P  # noqa: E402

p, k = int(sys.argv[1]), int(sys.argv[2])
d = P.SpatialDiscretization.build(p, k)
h = P.PMultigridHierarchy(d, 1e-4)
b1 = np.random.default_rng(1).standard_normal(d.n_free_1)
for _ in range(3):
    h.gauss_seidel_sweep(0, b1, b1)
