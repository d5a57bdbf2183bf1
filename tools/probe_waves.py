"""Per-wave kernel times of one profiled MGRIT solve (PHI_WAVE_DEBUG)."""
import os
import sys

import numpy as np

os.environ["PHI_WAVE_DEBUG"] = "1"
sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2107_05337_b200 as P  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
cfg = bench.CONFIGS[name]
d = P.SpatialDiscretization.build(cfg["p"], cfg["k"])
sol = P.MgritSolver(d, cfg["nt"], source_kind=cfg["source_kind"], source_param=cfg["source_param"],
                    init_kind=cfg["init_kind"], init_coeffs=bench.init_coeffs(cfg), cycle=cfg["cycle"], m=cfg["m"])
sol.solve()
sol.set_profile(True)
r = sol.solve()
print(sol.wave_report(), r.iterations)
