"""Developer probe for ncu: ILUT applications on the config-2 operator."""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2107_05337_b200 as P  # noqa: E402

d = P.SpatialDiscretization.build(3, 6)
h = P.PMultigridHierarchy(d, 1e-4, exact="exact" in sys.argv)
r = np.random.default_rng(0).standard_normal(d.n_free)
for _ in range(3):
    h.ilut_apply(r)
print("done")
