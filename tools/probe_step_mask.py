"""Developer probe: single-RHS Phi step (cluster path) wall time per developer mask."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2107_05337_b200 as P  # noqa: E402
from paper_2107_05337_b200 import engine as E  # noqa: E402

p, k = int(sys.argv[1]), int(sys.argv[2])
masks = [int(m) for m in sys.argv[3].split(",")] if len(sys.argv) > 3 else [0]
d = P.SpatialDiscretization.build(p, k)
st = E.ThetaStepper(d, 1.0, 8e-3, 1.0, E.default_solver_config(fixed_cycles=4))
u = np.random.default_rng(0).standard_normal((1, d.n_free))
for rep in range(2):
    for m in masks:
        E.dev_tuning(-m if m else 8, 8, 0)
        st.step(u)
        t = time.perf_counter()
        for _ in range(20):
            st.step(u)
        print(f"mask {m}: step (4 V-cycles) {1e3 * (time.perf_counter() - t) / 20:.3f} ms", flush=True)
