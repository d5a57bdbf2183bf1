"""Developer probe: wall time of the engine's single-CTA building blocks
(one kernel launch each, host-synchronised) to locate latency hot spots."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2107_05337_b200 as P  # noqa: E402

EXACT = "exact" in sys.argv


def t(fn, reps=5):
    fn()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    return (time.perf_counter() - t0) / reps * 1e3


def probe(p, k, c):
    d = P.SpatialDiscretization.build(p, k)
    h = P.PMultigridHierarchy(d, c, exact=EXACT)
    rng = np.random.default_rng(0)
    n, n1 = d.n_free, d.n_free_1
    r = rng.standard_normal(n)
    r1 = rng.standard_normal(n1)
    out = {
        "noop(spmv)": t(lambda: h.spmv(r)),
        "ilut": t(lambda: h.ilut_apply(r)),
        "restrict": t(lambda: h.restrict_to_linear(r)),
        "prolong": t(lambda: h.prolong_from_linear(r1)),
        "gs0": t(lambda: h.gauss_seidel_sweep(0, r1, r1)),
        "wcycle": t(lambda: h.hmg_wcycle(r1)),
        "vcycle": t(lambda: h.vcycle(r, np.zeros(n))),
        "solve": t(lambda: h.solve(r, None)),
    }
    print(f"p={p} k={k} n={n}: " + "  ".join(f"{k_}={v:.2f}ms" for k_, v in out.items()), flush=True)


if __name__ == "__main__":
    for p, k in [(2, 4), (3, 6)]:
        probe(p, k, 1e-4)
