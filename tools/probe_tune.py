"""Sweep the readiness-poll back-off on the single-CTA ILUT apply / W-cycle."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2107_05337_b200 as P  # noqa: E402
from paper_2107_05337_b200.engine import dev_tuning  # noqa: E402


def t(fn, reps=3):
    fn()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    return (time.perf_counter() - t0) / reps * 1e3


p, k = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (3, 6)
d = P.SpatialDiscretization.build(p, k)
h = P.PMultigridHierarchy(d, 1e-4)
r = np.random.default_rng(0).standard_normal(d.n_free)
r1 = np.random.default_rng(1).standard_normal(d.n_free_1)
for gw in (8,):
    for sl in (0,):
        dev_tuning(16, gw, sl)
        print(f"p={p} k={k} gs_warps={gw:2d} sleep={sl:4d}: ilut={t(lambda: h.ilut_apply(r)):8.3f} ms "
              f"gs0={t(lambda: h.gauss_seidel_sweep(0, r1, r1)):7.3f} ms "
              f"wcycle={t(lambda: h.hmg_wcycle(r1)):7.3f} ms vcycle={t(lambda: h.vcycle(r, 0*r)):7.3f} ms", flush=True)
