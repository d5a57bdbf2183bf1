"""CPU tests of the engine's host-side setup routines through the C ABI
(phi_setup_*, include/phi_engine.h): the quadrature / B-spline tables that feed
the device assembly, the dense coarse LU and the time-grid hierarchy rule,
bit for bit against fixtures made by the compiled reference
(tests/golden/setup_host.npz, tests/golden/make_golden.py) and, where
oracle/_ref is present, against the reference itself on further shapes.

Reference: quadrature.hpp:17-44, spline.hpp:48-63 and 104-130,
assembly.hpp:124-151 (detail::DirTables), solvers.hpp:102-172 (DenseLU),
mgrit.hpp:217-233 (build_levels), tests/test_mgrit.cpp:40-81."""
from __future__ import annotations

import os

import numpy as np
import pytest

import paper_2107_05337_b200 as P
from oracle import oracle as O
from paper_2107_05337_b200 import engine as E

from .golden import make_golden as G

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "setup_host.npz")


@pytest.fixture(scope="module")
def gold():
    P.lib()
    return np.load(GOLD)


def _same_bits(a, b) -> bool:
    a, b = np.ascontiguousarray(a), np.ascontiguousarray(b)
    return a.shape == b.shape and a.dtype == b.dtype and a.tobytes() == b.tobytes()


@pytest.mark.parametrize("case", G.SETUP_TABLE_CASES, ids=lambda c: "p%d_nel%d_nq%d" % c)
def test_tables_equal_the_reference_fixture(gold, case):
    p, nel, nq = case
    got = E.setup_tables_1d(p, nel, nq)
    for key, arr in got.items():
        assert _same_bits(arr, gold[f"t_{p}_{nel}_{nq}_{key}"]), (case, key)


def test_tables_are_a_partition_of_unity_and_integrate_exactly(gold):
    # known answers (the reference's tests/test_spline.cpp, test_quadrature.cpp properties)
    for p, nel, nq in [(2, 16, 3), (5, 256, 6), (1, 2, 2)]:
        t = E.setup_tables_1d(p, nel, nq)
        assert np.allclose(t["vals"].sum(axis=1), 1.0, rtol=0, atol=1e-14)
        assert np.allclose(t["ders"].sum(axis=1), 0.0, rtol=0, atol=1e-9 * nel)
        assert abs(t["weights"].sum() - 1.0) < 1e-14
        # an n-point rule integrates x^(2n-1) exactly over every span
        deg = 2 * nq - 1
        assert abs((t["weights"] * t["nodes"] ** deg).sum() - 1.0 / (deg + 1)) < 1e-14
        assert np.array_equal(t["first"], np.arange(nel))


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built (needs /root/reference)")
@pytest.mark.parametrize("p", [1, 2, 3, 4, 5, 6])
def test_tables_equal_the_compiled_reference(p):
    P.lib()
    for nel in (1, 2, 5, 8, 17, 32, 100):
        for nq in (p + 1, 2, 7):
            got, ref = E.setup_tables_1d(p, nel, nq), O.ref_tables_1d(p, nel, nq)
            for key in got:
                assert _same_bits(got[key], ref[key]), (p, nel, nq, key)


def test_dense_lu_solves_equal_the_reference_fixture(gold):
    inputs = G.setup_lu_inputs()
    for i, (a, b) in enumerate(inputs):
        assert _same_bits(a, gold[f"lu{i}_a"]) and _same_bits(b, gold[f"lu{i}_b"])  # the seeded inputs
        lu, piv = E.setup_dense_lu(a)
        assert sorted(piv.tolist()) == list(range(len(b)))
        x = O.lu_substitute(lu, piv, b)
        assert _same_bits(x, gold[f"lu{i}_x"]), i
        assert np.allclose(a @ x, b, atol=1e-9)


def test_dense_lu_pivots_on_the_first_largest_entry():
    P.lib()
    a = np.array([[0.0, 2.0, 1.0], [-3.0, 1.0, 0.0], [3.0, 0.0, 1.0]])
    lu, piv = E.setup_dense_lu(a)
    assert piv.tolist()[0] == 1  # |-3| ties |3|: the first one wins
    low = np.tril(lu, -1) + np.eye(3)
    assert np.allclose(low @ np.triu(lu), a[piv])


def test_dense_lu_errors_mirror_the_reference():
    P.lib()
    with pytest.raises(E.EngineError, match="DenseLU: singular matrix"):  # std::runtime_error
        E.setup_dense_lu(np.zeros((2, 2)))
    with pytest.raises(ValueError, match="DenseLU: matrix not square"):
        E.setup_dense_lu(np.zeros((2, 3)))
    with pytest.raises(ValueError, match="gauss_legendre_01: n must be >= 1"):
        E.setup_tables_1d(2, 4, 0)
    with pytest.raises(ValueError, match="open_uniform_knots: degree must be >= 1"):
        E.setup_tables_1d(0, 4, 2)
    with pytest.raises(ValueError, match="open_uniform_knots: n_elements must be >= 1"):
        E.setup_tables_1d(2, 0, 3)


def test_time_grid_hierarchy_rule():
    P.lib()
    # tests/test_mgrit.cpp:40-81
    assert E.setup_level_steps(16, 2, P.CYCLE_V, 2) == [16, 8, 4, 2]
    assert E.setup_level_steps(16, 16, P.CYCLE_V, 8) == [16, 1]
    assert E.setup_level_steps(256, 2, P.CYCLE_V, 8) == [256, 128, 64, 32, 16, 8]
    with pytest.raises(ValueError, match=r"MGRIT: nt \(100\) not divisible by coarsening factor m \(3\)"):
        E.setup_level_steps(100, 3, P.CYCLE_V, 8)
    with pytest.raises(ValueError, match="MgritConfig: m must be >= 2"):
        E.setup_level_steps(100, 1, P.CYCLE_V, 8)
    # fewer steps than m: a single level (tests/test_mgrit.cpp:252)
    assert E.setup_level_steps(3, 4, P.CYCLE_V, 8) == [3]
    # BASELINE configs: C2 two-level, C3 as the reference builds it, the divisible variants
    assert E.setup_level_steps(1000, 8, P.CYCLE_TWO_LEVEL, 8) == [1000, 125]
    assert E.setup_level_steps(2500, 4, P.CYCLE_V, 8) == [2500, 625]
    assert E.setup_level_steps(2560, 4, P.CYCLE_V, 100) == [2560, 640, 160]
    assert E.setup_level_steps(10240, 8, P.CYCLE_F, 8) == [10240, 1280, 160, 20]
    assert E.setup_level_steps(64, 2, P.CYCLE_F, 8) == [64, 32, 16, 8]
