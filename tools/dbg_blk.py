"""Developer check of the block sweeps on a small hierarchy (fast mode)."""
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_2107_05337_b200 as P

P.lib().phi_set_device(0)
p, k = int(sys.argv[1]), int(sys.argv[2])
disc = P.SpatialDiscretization.build(p, k)
h = P.PMultigridHierarchy(disc, 1e-3)
n = disc.n_free
r = np.random.default_rng(0).standard_normal(n)
b1 = np.random.default_rng(1).standard_normal(disc.n_free_1)
for name, f in [("spmv", lambda: h.spmv(r)), ("ilut", lambda: h.ilut_apply(r)),
                ("gs0", lambda: h.gauss_seidel_sweep(0, b1, b1)),
                ("gs0b", lambda: h.gauss_seidel_sweep(0, b1, b1, backward=True)),
                ("wcycle", lambda: h.hmg_wcycle(b1)), ("vcycle", lambda: h.vcycle(r, np.zeros(n)))]:
    print(name, "...", flush=True)
    z = f()
    print(name, "done", np.linalg.norm(z), flush=True)
