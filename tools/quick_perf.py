"""Developer timing probe (not the bench): MGRIT C1/C2 solve time and C5-style
batched V-cycles through the engine, CUDA-event timed where possible."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2107_05337_b200 as P  # noqa: E402


def mgrit(p, k, nt, m, **kw):
    d = P.SpatialDiscretization.build(p, k)
    t0 = time.time()
    g = P.MgritSolver(d, nt, m=m, cycle=P.CYCLE_TWO_LEVEL, **kw)
    t1 = time.time()
    r = g.solve()
    t2 = time.time()
    r = g.solve()
    t3 = time.time()
    print(f"p={p} k={k} nt={nt} n={d.n_free}: setup {t1-t0:.2f}s solve {t2-t1:.3f}s / {t3-t2:.3f}s "
          f"iters={r.iterations} solves={r.total_spatial_solves} mean={r.mean_spatial_iterations:.4f} "
          f"launches={g.launches()} dof*steps/s={d.n_free*nt/(t3-t2):.3e}", flush=True)


def vcyc(p, k, nrhs, c=1e-4):
    d = P.SpatialDiscretization.build(p, k)
    h = P.PMultigridHierarchy(d, c)
    rng = np.random.default_rng(0)
    b = rng.standard_normal((nrhs, d.n_free))
    x = np.zeros_like(b)
    h.vcycle(b, x)
    t0 = time.time()
    for _ in range(3):
        h.vcycle(b, x)
    t = (time.time() - t0) / 3
    print(f"vcycle p={p} k={k} B={nrhs}: {t*1e3:.2f} ms (incl. H2D/D2H)", flush=True)


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "all"
    if what in ("all", "c1"):
        mgrit(2, 4, 100, 4, source_param=0.0, init_kind=P.INIT_SIN)
    if what in ("all", "c2"):
        n = (2 ** 6 + 3 - 2) ** 2
        mgrit(3, 6, 1000, 8, source_kind=P.SOURCE_SIN_EXP, source_param=2 * np.pi ** 2,
              init_kind=P.INIT_COEFFS, init_coeffs=np.random.default_rng(12345).uniform(-1, 1, n))
    if what in ("all", "c5"):
        for p in (2, 5):
            for B in (1, 16, 64):
                vcyc(p, 8, B)
