"""The coarse march overlapped with the interpolation and the residual
(Mgrit::coarse_overlapped): the fine-level work of every interval runs on a
side stream as soon as the march has published both of its C-points.  It
performs the same operations per point as the serial phases, so the solve
must be bit-identical to the one with the overlap switched off
(PHI_OVERLAP=0): iterations, residual history, counts, trajectory."""
import os

import numpy as np
import pytest

from tests.conftest import gpu_available

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]

E = pytest.importorskip("paper_2107_05337_b200.engine")


def _solve(overlap, p, k, nt, **kw):
    os.environ["PHI_OVERLAP"] = "1" if overlap else "0"
    try:
        s = E.MgritSolver(E.SpatialDiscretization.build(p, k), nt, **kw)
    finally:
        os.environ.pop("PHI_OVERLAP", None)
    r = s.solve()
    return r, s.trajectory()


@pytest.mark.parametrize("case", [
    # two-level (the config-2 shape, 64 intervals): overlap with interpolation and residual
    dict(p=3, k=5, nt=512, cycle=E.CYCLE_TWO_LEVEL, m=8, source_kind=E.SOURCE_SIN_EXP,
         source_param=2 * np.pi ** 2, init_kind=E.INIT_SIN),
    # V-cycle over three levels (2048/512/128, as c3ml): overlap with level 1's interpolation
    dict(p=2, k=3, nt=2048, cycle=E.CYCLE_V, m=4, coarse_floor=41, source_param=1.0, init_kind=E.INIT_SIN),
    # F-cycle over three levels (256/128/64): the second pass re-enters the overlapped coarse cycle
    dict(p=2, k=3, nt=256, cycle=E.CYCLE_F, m=2, coarse_floor=33, source_kind=E.SOURCE_SIN, source_param=1.0),
])
def test_overlap_bit_identical(case):
    case = dict(case)
    p, k, nt = case.pop("p"), case.pop("k"), case.pop("nt")
    r0, t0 = _solve(False, p, k, nt, **case)
    r1, t1 = _solve(True, p, k, nt, **case)
    assert r1.iterations == r0.iterations and r1.converged == r0.converged
    assert np.array_equal(r1.residual_history, r0.residual_history)
    assert r1.total_spatial_solves == r0.total_spatial_solves
    assert r1.mean_spatial_iterations == r0.mean_spatial_iterations
    assert np.array_equal(t1, t0)
