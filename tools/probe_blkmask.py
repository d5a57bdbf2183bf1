"""Developer probe: ILUT apply (unit op 1) per-block cycles under developer masks."""
import ctypes as C
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2107_05337_b200 as P  # noqa: E402
from paper_2107_05337_b200 import engine as E  # noqa: E402

p, k = int(sys.argv[1]), int(sys.argv[2])
d = P.SpatialDiscretization.build(p, k)
h = P.PMultigridHierarchy(d, 1e-4)
b = np.random.default_rng(0).standard_normal(d.n_free)
nb = (d.n_free + 31) // 32
for m in (0, 2, 4, 8, 14):
    E.lib().phi_dev_tuning(-m if m else 8, 8, -1)
    h.ilut_apply(b)
    buf = np.zeros(49152, np.int64)
    E.lib().phi_dev_trace(buf.ctypes.data_as(C.c_void_p), buf.size)
    t = buf[24000:24000 + 8 * nb].reshape(nb, 8)
    print(f"mask {m:2d}: per block {np.median(np.diff(t[:, 3])):6.0f}  chain {np.median(t[:, 3] - t[:, 2]):6.0f} "
          f"cntwait {np.median(t[:, 1] - t[:, 0]):6.0f} pre {np.median(t[:, 2] - t[:, 1]):6.0f}", flush=True)
