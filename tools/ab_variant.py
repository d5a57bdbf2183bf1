"""Developer A/B of a library variant (PHI_VARIANT=<name> selects _lib_<name>):
timed solves of a bench config without the profile, and a hash of the
trajectory so that two builds can be compared bit for bit.

    [PHI_VARIANT=tri] python tools/ab_variant.py c2 3      # 3 full solves
    [PHI_VARIANT=tri] python tools/ab_variant.py c3 2 1    # 2 x (initialize + 1 cycle)
"""
import hashlib
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2107_05337_b200 as P  # noqa: E402
from paper_2107_05337_b200 import engine as E  # noqa: E402


def main():
    name, reps = sys.argv[1], int(sys.argv[2])
    iters = int(sys.argv[3]) if len(sys.argv) > 3 else 0
    cfg = dict(bench.CONFIGS[name])
    E.lib().phi_set_device(0)
    disc = P.SpatialDiscretization.build(cfg["p"], cfg["k"])
    sol = P.MgritSolver(disc, cfg["nt"], source_kind=cfg["source_kind"], source_param=cfg["source_param"],
                        init_kind=cfg["init_kind"], init_coeffs=bench.init_coeffs(cfg), cycle=cfg["cycle"],
                        m=cfg["m"], coarse_floor=cfg.get("coarse_floor", 8))
    times, info = [], None
    for _ in range(reps + 1):  # the first one warms up
        E.lib().phi_synchronize()
        t0 = time.perf_counter()
        if iters == 0:
            r = sol.solve()
            info = (r.iterations, r.total_spatial_solves)
        else:
            sol.initialize()
            for _ in range(iters):
                sol.mgrit_cycle(0)
            info = sol.residual_norm(0)
        E.lib().phi_synchronize()
        times.append(time.perf_counter() - t0)
    digest = hashlib.sha256(sol.trajectory().tobytes()).hexdigest()[:16]
    print(json.dumps({"variant": os.environ.get("PHI_VARIANT", ""), "config": name, "iters": iters,
                      "seconds": times[1:], "info": info, "trajectory_sha": digest}), flush=True)


if __name__ == "__main__":
    main()
