"""Developer helper for ncu captures: one SpMV / SpMM launch set at a config-5
shape.  python tools/c5_one.py p B"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2107_05337_b200 as P  # noqa: E402
from paper_2107_05337_b200 import engine as E  # noqa: E402

p, b = int(sys.argv[1]), int(sys.argv[2])
E.lib().phi_set_device(0)
d = P.SpatialDiscretization.build(p, 8)
h = P.PMultigridHierarchy(d, 1e-4)
print(p, b, h.time_kernel(0, b, reps=2, flush_l2=1))
