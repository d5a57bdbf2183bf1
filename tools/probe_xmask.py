"""Developer probe: ILUT / W-cycle / V-cycle times under timing experiments
(phi_dev_tuning(-mask, ..)): 1 = no butterfly, 2 = no z loads."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2107_05337_b200 as P  # noqa: E402
from paper_2107_05337_b200 import engine as E  # noqa: E402

d = P.SpatialDiscretization.build(3, 6)
h = P.PMultigridHierarchy(d, 1e-4)
r = np.random.default_rng(0).standard_normal(d.n_free)
r1 = np.random.default_rng(1).standard_normal(d.n_free_1)


def t(fn, reps=5):
    fn()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    return (time.perf_counter() - t0) / reps * 1e3


for mask in (0, 1, 2, 3):
    E.lib().phi_dev_tuning(-mask if mask else 0, 8, 0)
    print(f"mask {mask}: ilut {t(lambda: h.ilut_apply(r)):.3f} ms  wcycle {t(lambda: h.hmg_wcycle(r1)):.3f} ms  "
          f"noop {t(lambda: h.spmv(r)):.3f} ms", flush=True)
