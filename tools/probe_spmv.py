"""Developer probe: one SpMV / SpMM of config 5 (p, B) for ncu."""
import sys

sys.path.insert(0, ".")
import paper_2107_05337_b200 as P  # noqa: E402

p, b = int(sys.argv[1]), int(sys.argv[2])
d = P.SpatialDiscretization.build(p, 8)
h = P.PMultigridHierarchy(d, 1e-4)
print(h.time_kernel(0, b, reps=3))
