"""Device ILUT factorisation (csrc/ilut.cu) against the reference's
ilut_factor (ilut.hpp:29-143) compiled here (oracle/_ref): the L and U
factors must be bit-identical -- same kept entries (keep_largest,
ilut.hpp:112-124), same columns, same values -- at the BASELINE operator
shapes and under the reference's own ILUT test regimes
(tests/test_linalg.cpp:140-243: tau = 0 with full fill is the exact LU,
fill limits, drop tolerances)."""
import numpy as np
import pytest

from oracle import oracle as O
from tests.conftest import gpu_available

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]

E = pytest.importorskip("paper_2107_05337_b200.engine")


def _same(a, b, what):
    assert (a.n_rows, a.n_cols) == (b.n_rows, b.n_cols), what
    assert np.array_equal(a.row_offsets, b.row_offsets), what
    assert np.array_equal(a.col_indices, b.col_indices), what
    assert np.array_equal(a.values, b.values), (what, np.max(np.abs(a.values - b.values)))


def _check(p, k, c, tau=1e-13, fill=0):
    if not O.ref_available():
        pytest.skip("oracle/_ref not built (make -C oracle ref)")
    d = E.SpatialDiscretization.build(p, k)
    h = E.PMultigridHierarchy(d, c, ilut_tau=tau, ilut_fill=fill)
    r = O.RefHier(O.RefDisc(p, k), c, tau=tau, fill=fill)
    _same(h.csr(0), r.csr(0), "A")
    _same(h.csr(1), r.csr(1), "L")
    _same(h.csr(2), r.csr(2), "U")


@pytest.mark.parametrize("p,k,c", [(2, 4, 1e-3), (3, 6, 1e-4), (3, 6, 8e-4), (1, 5, 1e-2), (6, 4, 1e-3)])
def test_device_ilut_bitwise(p, k, c):
    """config 1 and 2 operators (both MGRIT levels), degree 1 and 6."""
    _check(p, k, c)


@pytest.mark.parametrize("tau,fill", [(0.0, 10_000), (1e-3, 0), (1e-13, 5), (0.1, 3)])
def test_device_ilut_regimes(tau, fill):
    """exact LU (tau 0, unlimited fill), heavy dropping, tight fill limits
    (many ties broken by column)."""
    _check(2, 4, 1e-3, tau=tau, fill=fill)


@pytest.mark.slow
@pytest.mark.parametrize("p,k,c", [(4, 7, 4e-5), (5, 8, 1e-5)])
def test_device_ilut_bitwise_large(p, k, c):
    """config 3 (p=4, h=2^-7) and config 4 (p=5, h=2^-8) level-0 operators."""
    _check(p, k, c)
