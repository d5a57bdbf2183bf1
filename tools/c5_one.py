"""Developer helper for ncu captures: one SpMV / SpMM launch set at a config-5
shape, or (third argument 1) one V(1,1) cycle.  python tools/c5_one.py p B [which]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2107_05337_b200 as P  # noqa: E402
from paper_2107_05337_b200 import engine as E  # noqa: E402

p, b = int(sys.argv[1]), int(sys.argv[2])
E.lib().phi_set_device(0)
d = P.SpatialDiscretization.build(p, 8)
h = P.PMultigridHierarchy(d, 1e-4)
which = int(sys.argv[3]) if len(sys.argv) > 3 else 0
print(p, b, which, h.time_kernel(which, b, reps=2, flush_l2=1))
