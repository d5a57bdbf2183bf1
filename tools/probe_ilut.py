"""ncu target: a few single-CTA ILUT applications (L then U solve)."""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2107_05337_b200 as P  # noqa: E402
from paper_2107_05337_b200.engine import dev_tuning  # noqa: E402

p, k = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (3, 6)
warps = int(sys.argv[3]) if len(sys.argv) > 3 else 16
dev_tuning(warps, warps, 0)
d = P.SpatialDiscretization.build(p, k)
h = P.PMultigridHierarchy(d, 1e-4)
r = np.random.default_rng(0).standard_normal(d.n_free)
for _ in range(3):
    z = h.ilut_apply(r)
print("ok", float(np.abs(z).sum()))
