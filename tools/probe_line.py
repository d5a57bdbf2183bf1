"""Developer probe: per-line stamps of the line Gauss-Seidel chain (PHI_TRACE=1
build), level-0 forward sweep (unit op 5)."""
import ctypes as C
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2107_05337_b200 as P  # noqa: E402
from paper_2107_05337_b200 import engine as E  # noqa: E402

p, k = int(sys.argv[1]), int(sys.argv[2])
d = P.SpatialDiscretization.build(p, k)
h = P.PMultigridHierarchy(d, 1e-4)
b1 = np.random.default_rng(1).standard_normal(d.n_free_1)
h.gauss_seidel_sweep(0, b1, b1)
E.dev_tuning(8, 8, -1)
h.gauss_seidel_sweep(0, b1, b1)
buf = np.zeros(49152, np.int64)
E.lib().phi_dev_trace(buf.ctypes.data_as(C.c_void_p), buf.size)
nf = int(round(d.n_free_1 ** 0.5))
t = buf[24000:24000 + 8 * nf].reshape(nf, 8)
for name, v in {"loads->beta": t[:, 1] - t[:, 0], "scan": t[:, 2] - t[:, 1], "store": t[:, 3] - t[:, 2],
                "gap": np.r_[t[1:, 0] - t[:-1, 3], 0], "per line": np.r_[np.diff(t[:, 0]), 0]}.items():
    print(f"{name:12s} median {np.median(v):7.0f} mean {v.mean():7.0f} max {v.max():7.0f}")
