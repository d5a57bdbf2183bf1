"""Trace per-block clock64 stamps of the warp-pipelined triangular solve."""
import ctypes as C
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2107_05337_b200 as P  # noqa: E402
from paper_2107_05337_b200.engine import lib  # noqa: E402

d = P.SpatialDiscretization.build(3, 6)
h = P.PMultigridHierarchy(d, 1e-4)
r = np.random.default_rng(0).standard_normal(d.n_free)
h.ilut_apply(r)
lib().phi_dev_tuning(8, 8, -1)
h.ilut_apply(r)   # trace records the U solve (last writer wins per block slot)
buf = np.zeros(8 * 1024 * 6, np.int64)
lib().phi_dev_trace.argtypes = [C.c_void_p, C.c_int]
lib().phi_dev_trace(buf.ctypes.data, buf.size)
t = buf[:8 * 1024 * 2].reshape(8, 1024, 2)
t0 = t[t > 0].min()
for w in range(3):
    row = t[w]
    nz = row[:, 0] > 0
    st = row[nz, 0] - t0
    en = row[nz, 1] - t0
    print(f"warp {w}: blocks={nz.sum()} first={st[:6]} dur={ (en-st)[:12]}")
    print("   gaps between blocks:", np.diff(st)[:20])
allst = t[:, :, 0][t[:, :, 0] > 0] - t0
allen = t[:, :, 1][t[:, :, 0] > 0] - t0
print("span cycles", allen.max(), "blocks", allst.size, "mean block dur", float(np.mean(allen - allst)),
      "median", float(np.median(allen - allst)))
