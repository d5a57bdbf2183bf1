"""Per-wavefront clock64 stamps of the barrier-synchronous Gauss-Seidel sweep."""
import ctypes as C
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2107_05337_b200 as P  # noqa: E402
from paper_2107_05337_b200.engine import lib  # noqa: E402

p, k = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (3, 6)
d = P.SpatialDiscretization.build(p, k)
h = P.PMultigridHierarchy(d, 1e-4)
r1 = np.random.default_rng(1).standard_normal(d.n_free_1)
h.gauss_seidel_sweep(0, r1, r1)
lib().phi_dev_tuning(8, 8, -1)
h.gauss_seidel_sweep(0, r1, r1)
buf = np.zeros(8 * 1024 * 6, np.int64)
lib().phi_dev_trace.argtypes = [C.c_void_p, C.c_int]
lib().phi_dev_trace(buf.ctypes.data, buf.size)
g = buf[8 * 1024 * 2:8 * 1024 * 2 + 4096].reshape(1024, 4)
nz = g[:, 0] > 0
g = g[nz]
print("wavefronts", len(g))
print("first row", np.median(g[:, 1] - g[:, 0]), " extra rows", np.median(g[:, 2] - g[:, 1]),
      " syncwarp", np.median(g[:, 3] - g[:, 2]), " -> next start", np.median(g[1:, 0] - g[:-1, 3]),
      " per wavefront", np.median(g[1:, 0] - g[:-1, 0]))
print("first rows:", (g[:6] - g[0, 0]).tolist())
