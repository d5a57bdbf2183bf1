"""Developer probe: per-cycle cost inside the fused wave kernel (solve with
fixed cycles) vs the standalone V-cycle kernel, same hierarchy."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2107_05337_b200 as P  # noqa: E402

EXACT = "exact" in sys.argv


def t(fn, reps=3):
    fn()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    return (time.perf_counter() - t0) / reps * 1e3


for (p, k, c) in [(3, 6, 1e-4), (3, 6, 8e-4)]:
    d = P.SpatialDiscretization.build(p, k)
    h = P.PMultigridHierarchy(d, c, exact=EXACT)
    b = np.random.default_rng(0).standard_normal(d.n_free)
    out = {"vcycle": t(lambda: h.vcycle(b, np.zeros(d.n_free)))}
    for fc in (1, 2, 4):
        out[f"solve_fc{fc}"] = t(lambda: h.solve(b, None, fixed_cycles=fc))
    print(f"p={p} k={k} c={c}: " + "  ".join(f"{a}={v:.2f}ms" for a, v in out.items()), flush=True)
