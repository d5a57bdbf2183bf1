"""Developer driver: one ILUT apply (unit op 1) for ncu."""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2107_05337_b200 as P  # noqa: E402

p, k = int(sys.argv[1]), int(sys.argv[2])
d = P.SpatialDiscretization.build(p, k)
h = P.PMultigridHierarchy(d, 1e-4)
b = np.random.default_rng(1).standard_normal(d.n_free)
for _ in range(3):
    h.ilut_apply(b)
