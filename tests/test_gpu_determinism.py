"""Run-to-run determinism of the hand-off protocols (compute-sanitizer is
closed on this pool, so races are hunted by repetition): the block-sweep
workers and solvers hand data over through shared-memory flags with
release/acquire semantics, the single-RHS waves run on clusters with DSMEM,
the rolling-window streams overwrite a shared ring.  A race would show up as
a result that changes between identical runs; every run here must be
bit-identical to the first."""
import numpy as np
import pytest

from tests.conftest import gpu_available

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]

E = pytest.importorskip("paper_2107_05337_b200.engine")


@pytest.mark.parametrize("p,k,nt,m", [(3, 6, 64, 8), (4, 7, 16, 4)])
def test_repeated_solves_bit_identical(p, k, nt, m):
    """(3, 6): z in shared memory, clusters for the coarse march; (4, 7): the
    rolling-window ILUT streams (z global)."""
    coeffs = np.random.default_rng(12345).uniform(-1, 1, (2 ** k + p - 2) ** 2)
    s = E.MgritSolver(E.SpatialDiscretization.build(p, k), nt, cycle=E.CYCLE_TWO_LEVEL, m=m,
                      source_kind=E.SOURCE_SIN_EXP, source_param=2 * np.pi ** 2, init_kind=E.INIT_COEFFS,
                      init_coeffs=coeffs)
    r0 = s.solve()
    t0 = s.trajectory()
    for _ in range(4):
        r = s.solve()
        assert r.iterations == r0.iterations
        assert np.array_equal(r.residual_history, r0.residual_history)
        assert np.array_equal(s.trajectory(), t0)


def test_repeated_batched_vcycles_bit_identical():
    """Many right-hand sides per wave (one CTA each, all SMs busy)."""
    d = E.SpatialDiscretization.build(3, 6)
    h = E.PMultigridHierarchy(d, 1e-4)
    B = np.random.default_rng(3).standard_normal((300, d.n_free))
    X0 = h.vcycle(B, np.zeros_like(B))
    for _ in range(3):
        assert np.array_equal(h.vcycle(B, np.zeros_like(B)), X0)
