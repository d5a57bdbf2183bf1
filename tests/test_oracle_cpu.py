"""CPU tests of the parity oracle (no GPU).

1. Known-answer tests of the reference's own suite for this path, re-expressed
   on the C restatement (oracle/phi_oracle.c):
   spmv            tests/test_linalg.cpp:33-64
   Gauss-Seidel    tests/test_linalg.cpp:101-138
   ILUT            tests/test_linalg.cpp:140-243
   transfers       tests/test_pmultigrid.cpp:12-34
   V-cycle         tests/test_pmultigrid.cpp:127-174
2. The restatement pinned bit for bit against golden fixtures produced by the
   compiled reference (tests/golden/make_golden.py).
3. When oracle/_ref is built here, the fixtures are re-derived from it.
"""
from __future__ import annotations

import os
import subprocess

import numpy as np
import pytest

from oracle import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")


@pytest.fixture(scope="module", autouse=True)
def _oracle_built():
    if not os.path.exists(O.OC_SO):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)


def _gold(name):
    return np.load(os.path.join(GOLD, name))


def _csr(g, prefix) -> O.CSR:
    nr, nc = (int(v) for v in g[prefix + "_shape"])
    return O.CSR(nr, nc, g[prefix + "_ro"], g[prefix + "_ci"], g[prefix + "_v"])


def _ops(g) -> dict:
    nh = int(g["n_h"][0])
    return {"mass_p": _csr(g, "mass_p"), "stiff_p": _csr(g, "stiff_p"), "transfer": _csr(g, "transfer"),
            "inv_lumped_p": g["inv_lumped_p"], "inv_lumped_1": g["inv_lumped_1"],
            "h_mass": [_csr(g, f"h_mass{l}") for l in range(nh)],
            "h_stiff": [_csr(g, f"h_stiff{l}") for l in range(nh)],
            "h_embed": [_csr(g, f"h_embed{l}") for l in range(nh - 1)]}


def _dense_csr(a: np.ndarray) -> O.CSR:
    ro, ci, v = [0], [], []
    for i in range(a.shape[0]):
        for j in range(a.shape[1]):
            if a[i, j] != 0.0:
                ci.append(j)
                v.append(a[i, j])
        ro.append(len(ci))
    return O.CSR(a.shape[0], a.shape[1], np.array(ro, np.int32), np.array(ci, np.int32), np.array(v))


def _same_csr(a: O.CSR, b: O.CSR) -> None:
    assert (a.n_rows, a.n_cols) == (b.n_rows, b.n_cols)
    assert np.array_equal(a.row_offsets, b.row_offsets)
    assert np.array_equal(a.col_indices, b.col_indices)
    assert np.array_equal(a.values, b.values)


# ---- known answers (reference test suite) ---------------------------------
def test_spmv_kat():
    a = _dense_csr(np.array([[4.0, 1.0], [1.0, 3.0]]))
    assert O.oc_spmv(a, np.array([1.0, 2.0])).tolist() == [6.0, 7.0]
    eye = _dense_csr(np.eye(4))
    x = np.array([1.0, -2.0, 3.5, 0.25])
    assert np.array_equal(O.oc_spmv(eye, x), x)
    assert np.array_equal(O.oc_spmv_transpose(a, np.array([1.0, 2.0])), np.array([6.0, 7.0]))


def test_spmv_distributes_and_matches_numpy():
    g = _gold("ops_p2k3.npz")
    a = _csr(g, "A")
    rng = np.random.default_rng(21)
    for _ in range(5):
        x, y = rng.uniform(-1, 1, a.n_cols), rng.uniform(-1, 1, a.n_cols)
        lhs = O.oc_spmv(a, x + y)
        np.testing.assert_allclose(lhs, O.oc_spmv(a, x) + O.oc_spmv(a, y), atol=1e-14)
        assert np.array_equal(O.oc_spmv(a, x), a.spmv(x))  # same sequential row order


def test_gauss_seidel_kat():
    d = _dense_csr(np.diag([2.0, 4.0, 0.5]))
    assert O.oc_gs_sweep(d, np.array([2.0, 8.0, 1.0]), np.zeros(3)).tolist() == [1.0, 2.0, 2.0]
    a = _dense_csr(np.array([[2.0, 1.0], [1.0, 2.0]]))
    assert O.oc_gs_sweep(a, np.array([3.0, 3.0]), np.zeros(2)).tolist() == [1.5, 0.75]
    with pytest.raises(RuntimeError):
        O.oc_gs_sweep(_dense_csr(np.array([[0.0, 1.0], [1.0, 0.0]])), np.ones(2), np.zeros(2))


def test_gauss_seidel_fixed_point():
    g = _gold("ops_p2k3.npz")
    a = _csr(g, "a_h0")
    xs = np.random.default_rng(9).uniform(-1, 1, a.n_rows)
    b = O.oc_spmv(a, xs)
    np.testing.assert_allclose(O.oc_gs_sweep(a, b, xs), xs, atol=1e-12)
    np.testing.assert_allclose(O.oc_gs_sweep(a, b, xs, backward=True), xs, atol=1e-12)


def test_ilut_full_fill_is_exact_lu():
    g = _gold("ops_p2k3.npz")
    disc = O.OcDisc(_ops(g))
    n = disc.n
    h = O.OcHier(disc, 0.05, tau=0.0, fill=n)
    lo, up = h.csr(1).dense(), h.csr(2).dense()
    a = h.csr(0).dense()
    lu = (lo + np.eye(n)) @ up
    assert np.abs(lu - a).sum(1).max() / np.abs(a).sum(1).max() <= 1e-12
    # exact factors: ilut_apply is the inverse (tests/test_linalg.cpp:220-229)
    b = np.random.default_rng(3).uniform(-1, 1, n)
    np.testing.assert_allclose(O.oc_spmv(h.csr(0), h.ilut_apply(b)), b, atol=1e-11)


def test_ilut_deterministic_and_linear():
    g = _gold("ops_p2k3.npz")
    disc = O.OcDisc(_ops(g))
    h1, h2 = O.OcHier(disc, 0.02, tau=1e-3, fill=5), O.OcHier(disc, 0.02, tau=1e-3, fill=5)
    _same_csr(h1.csr(1), h2.csr(1))
    _same_csr(h1.csr(2), h2.csr(2))
    assert max(np.diff(h1.csr(1).row_offsets)) <= 5 and max(np.diff(h1.csr(2).row_offsets)) <= 6
    rng = np.random.default_rng(5)
    x, y = rng.uniform(-1, 1, disc.n), rng.uniform(-1, 1, disc.n)
    np.testing.assert_allclose(h1.ilut_apply(2.0 * x + y), 2.0 * h1.ilut_apply(x) + h1.ilut_apply(y),
                               rtol=1e-12, atol=1e-12)


def test_transfers_and_vcycle_properties():
    g = _gold("ops_p2k3.npz")
    disc = O.OcDisc(_ops(g))
    h = O.OcHier(disc, 1e-3)
    # prolong = (M^L_p)^-1 T e1, restrict = (M^L_1)^-1 T^T r (pmultigrid.hpp:240-254;
    # tests/test_pmultigrid.cpp:12-34)
    tr = _csr(g, "transfer")
    e1 = np.random.default_rng(1).uniform(-1, 1, disc.n1)
    assert np.array_equal(h.prolong(e1), O.oc_spmv(tr, e1) * g["inv_lumped_p"])
    r = np.random.default_rng(2).uniform(-1, 1, disc.n)
    assert np.array_equal(h.restrict(r), O.oc_spmv_transpose(tr, r) * g["inv_lumped_1"])
    np.testing.assert_allclose(h.restrict(3.0 * r), 3.0 * h.restrict(r), rtol=1e-14, atol=1e-15)
    # V-cycle: the exact solution is a fixed point (127-138); homogeneity (159-174)
    a = h.csr(0)
    xs = np.random.default_rng(4).uniform(-1, 1, disc.n)
    b = O.oc_spmv(a, xs)
    np.testing.assert_allclose(h.vcycle(b, xs), xs, atol=1e-12)
    np.testing.assert_allclose(h.vcycle(2.0 * b, np.zeros(disc.n)), 2.0 * h.vcycle(b, np.zeros(disc.n)),
                               rtol=1e-12, atol=1e-13)
    # contraction <= 0.5 (140-157)
    x = np.zeros(disc.n)
    e0 = np.linalg.norm(xs - x)
    x = h.vcycle(b, x)
    assert np.linalg.norm(xs - x) <= 0.5 * e0


# ---- pinned against the compiled reference (golden fixtures) ---------------
def test_restatement_matches_reference_building_blocks():
    g = _gold("ops_p2k3.npz")
    disc = O.OcDisc(_ops(g))
    h = O.OcHier(disc, float(g["c"][0]))
    _same_csr(h.csr(0), _csr(g, "A"))
    _same_csr(h.csr(1), _csr(g, "L"))
    _same_csr(h.csr(2), _csr(g, "U"))
    assert np.array_equal(h.ilut_apply(g["b"]), g["ilut_apply"])
    assert np.array_equal(h.restrict(g["b"]), g["restrict"])
    assert np.array_equal(h.prolong(g["b1"]), g["prolong"])
    assert np.array_equal(h.hmg_wcycle(g["b1"]), g["wcycle"])
    a0 = _csr(g, "a_h0")
    assert np.array_equal(O.oc_gs_sweep(a0, g["b1"], g["x1"]), g["gs_fwd"])
    assert np.array_equal(O.oc_gs_sweep(a0, g["b1"], g["x1"], backward=True), g["gs_bwd"])
    assert np.array_equal(h.coarse_solve(g["bc"]), g["coarse"])
    assert np.array_equal(h.vcycle(g["b"], np.zeros(disc.n)), g["vcycle"])
    s = h.solve(g["b"])
    assert s["iterations"] == int(g["solve_iters"][0])
    assert np.array_equal(s["x"], g["solve_x"])
    assert np.array_equal(s["residual_history"], g["solve_hist"])


@pytest.mark.parametrize("name,kw", [
    ("mgrit_c1.npz", dict(cycle=O.CYCLE_TWO_LEVEL, m=4)),
    ("mgrit_src.npz", dict(cycle=O.CYCLE_TWO_LEVEL, m=8)),
    ("mgrit_cg.npz", dict(cycle=O.CYCLE_TWO_LEVEL, m=8, spatial_kind=1)),
])
def test_restatement_matches_reference_mgrit(name, kw):
    g = _gold(name)
    ops = _ops(g)
    nt = g["trajectory"].shape[0] - 1
    loads = g["loads"] if "loads" in g.files else None
    oc = O.OcMgrit(O.OcDisc(ops), nt, u0=g["u0"], loads=loads, **kw)
    assert oc.levels()[0] == g["levels_steps"].tolist()
    r = oc.solve()
    assert r["iterations"] == int(g["iterations"][0])
    assert r["total_spatial_solves"] == int(g["solves"][0])
    assert r["mean_spatial_iterations"] == float(g["mean_iters"][0])
    assert np.array_equal(r["residual_history"], g["history"])
    assert np.array_equal(oc.trajectory(), g["trajectory"])


def test_fixtures_current():
    """Re-derive one fixture from the compiled reference when it is built here."""
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    import importlib.util

    spec = importlib.util.spec_from_file_location("make_golden", os.path.join(GOLD, "make_golden.py"))
    mg = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mg)
    fresh = mg.ops_fixture()
    g = _gold("ops_p2k3.npz")
    for key in ("L_v", "U_v", "ilut_apply", "vcycle", "solve_x"):
        assert np.array_equal(fresh[key], g[key]), key
