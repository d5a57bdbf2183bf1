"""Developer probe: single-RHS V-cycle wall time per developer mask."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2107_05337_b200 as P  # noqa: E402
from paper_2107_05337_b200 import engine as E  # noqa: E402

p, k = int(sys.argv[1]), int(sys.argv[2])
masks = [int(m) for m in sys.argv[3].split(",")] if len(sys.argv) > 3 else [0]
d = P.SpatialDiscretization.build(p, k)
h = P.PMultigridHierarchy(d, 1e-4)
b = np.random.default_rng(0).standard_normal(d.n_free)
x0 = np.zeros(d.n_free)
for m in masks:
    E.dev_tuning(-m if m else 8, 8, 0)
    h.vcycle(b, x0)
    t = time.perf_counter()
    for _ in range(20):
        h.vcycle(b, x0)
    print(f"mask {m}: vcycle {1e3 * (time.perf_counter() - t) / 20:.3f} ms", flush=True)
