"""Developer probe: where one MGRIT solve's device time goes, per wave kind.

    python tools/probe_breakdown.py c3 [iters]

Runs initialize() + `iters` MGRIT cycles (default: a full solve()) with the
per-wave CUDA-event profile on and prints, per level and wave size, the
summed kernel time.  Not the bench (see bench.py)."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2107_05337_b200 as P  # noqa: E402
from paper_2107_05337_b200 import engine as E  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c3"
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    cfg = dict(bench.CONFIGS[name])
    for kv in sys.argv[3:]:
        k, v = kv.split("=")
        cfg[k] = int(v)
    E.lib().phi_set_device(0)
    t0 = time.time()
    disc = P.SpatialDiscretization.build(cfg["p"], cfg["k"])
    sol = P.MgritSolver(disc, cfg["nt"], source_kind=cfg["source_kind"], source_param=cfg["source_param"],
                        init_kind=cfg["init_kind"], init_coeffs=bench.init_coeffs(cfg), cycle=cfg["cycle"],
                        m=cfg["m"], coarse_floor=cfg.get("coarse_floor", 8))
    print(f"setup {time.time() - t0:.1f} s, levels {sol.levels()}", flush=True)
    sol.set_profile(True)
    E.lib().phi_synchronize()
    t0 = time.time()
    if iters == 0:
        r = sol.solve()
        print(f"solve: {r.iterations} iterations, {r.total_spatial_solves} solves, "
              f"mean {r.mean_spatial_iterations:.4f}", flush=True)
    else:
        sol.initialize()
        for _ in range(iters):
            sol.mgrit_cycle(0)
            print("rel", sol.residual_norm(0), flush=True)
    E.lib().phi_synchronize()
    wall = time.time() - t0
    os.environ["PHI_WAVE_DEBUG"] = "1"
    nw, ms, by = sol.wave_report()
    print(json.dumps({"config": name, "wall_s": wall, "waves": nw, "wave_ms": ms, "bytes": by}), flush=True)


if __name__ == "__main__":
    main()
