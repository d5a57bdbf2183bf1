"""Developer probe for ncu: one V-cycle (vcycle_kernel) then one fixed-cycle
solve (phi_wave_kernel) on the config-2 operator."""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2107_05337_b200 as P  # noqa: E402

d = P.SpatialDiscretization.build(3, 6)
h = P.PMultigridHierarchy(d, 1e-4, exact=len(sys.argv) > 1 and sys.argv[1] == "exact")
b = np.random.default_rng(0).standard_normal(d.n_free)
h.vcycle(b, np.zeros(d.n_free))
h.solve(b, None, fixed_cycles=1)
print("done")
