"""GPU parity of the CG spatial-solver kind (SpatialSolverKind::cg, theta.hpp:64,
121-125): Phi solved by Jacobi-preconditioned CG (solvers.hpp:21-75) instead of
p-multigrid.

Exact mode: bit-identical to the C restatement (oracle/phi_oracle.c) and to the
golden fixture tests/golden/mgrit_cg.npz made by the compiled reference.
Default (reassociated) mode: the north-star tolerance -- iteration counts
within +-1, space-time solution within 1e-8 relative L2.
"""
import os

import numpy as np
import pytest

from oracle import oracle as O
from tests.conftest import gpu_available

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]

E = pytest.importorskip("paper_2107_05337_b200.engine")

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
TOL_TRAJ = 1e-8


def _cfg(exact, **kw):
    return E.default_solver_config(exact=int(exact), kind=E.SOLVER_CG, **kw)


def _rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.parametrize("nrhs", [1, 3])
def test_cg_step_bitwise(nrhs):
    d = E.SpatialDiscretization.build(3, 5)
    dt = 1e-3
    st = E.ThetaStepper(d, 1.0, dt, 1.0, _cfg(True))
    ost = O.OcStepper(O.OcDisc(d.operators()), 1.0, dt, 1.0, kind=1)
    rng = np.random.default_rng(29)
    u = rng.standard_normal((nrhs, d.n_free))
    load = rng.standard_normal((nrhs, d.n_free))
    guess = rng.standard_normal((nrhs, d.n_free))
    got = st.step(u, load, guess)
    for i in range(nrhs):
        ref, _ = ost.step(u[i], load[i], guess[i])
        assert np.array_equal(got[i], ref)


def _golden_case():
    g = np.load(os.path.join(GOLD, "mgrit_cg.npz"))
    kw = dict(cycle=E.CYCLE_TWO_LEVEL, m=8, source_kind=E.SOURCE_SIN_EXP,
              source_param=2 * np.pi ** 2, init_kind=E.INIT_COEFFS, init_coeffs=g["coeffs"])
    return g, kw


def test_cg_mgrit_bitwise_vs_golden():
    g, kw = _golden_case()
    d = E.SpatialDiscretization.build(3, 4)
    nt = g["trajectory"].shape[0] - 1
    eng = E.MgritSolver(d, nt, solver=_cfg(True), **kw)
    assert eng.levels()[0] == g["levels_steps"].tolist()
    r = eng.solve()
    assert r.iterations == int(g["iterations"][0])
    assert r.total_spatial_solves == int(g["solves"][0])
    assert r.mean_spatial_iterations == float(g["mean_iters"][0])
    assert np.array_equal(r.residual_history, g["history"])
    assert np.array_equal(eng.trajectory(), g["trajectory"])


def test_cg_mgrit_fast_within_tolerance():
    g, kw = _golden_case()
    d = E.SpatialDiscretization.build(3, 4)
    nt = g["trajectory"].shape[0] - 1
    eng = E.MgritSolver(d, nt, solver=_cfg(False), **kw)
    r = eng.solve()
    assert abs(r.iterations - int(g["iterations"][0])) <= 1
    assert abs(r.mean_spatial_iterations - float(g["mean_iters"][0])) <= 1.0
    assert _rel(eng.trajectory(), g["trajectory"]) <= TOL_TRAJ


def test_cg_fast_single_rhs_cluster_path():
    # one right-hand side runs on a cluster of CTAs in the default mode
    d = E.SpatialDiscretization.build(3, 6)
    dt = 1e-3
    st = E.ThetaStepper(d, 1.0, dt, 1.0, _cfg(False))
    ost = O.OcStepper(O.OcDisc(d.operators()), 1.0, dt, 1.0, kind=1)
    rng = np.random.default_rng(31)
    u = rng.standard_normal((1, d.n_free))
    got = st.step(u, None, None)
    ref, _ = ost.step(u[0], None, None)
    assert _rel(got[0], ref) <= 1e-10


def test_cg_not_converged_message():
    d = E.SpatialDiscretization.build(2, 4)
    st = E.ThetaStepper(d, 1.0, 1e-2, 1.0, _cfg(True, max_iter=2))
    u = np.random.default_rng(5).standard_normal((1, d.n_free))
    with pytest.raises(Exception, match=r"spatial solve did not converge \(cg\)"):
        st.step(u, None, None)


def test_cg_theta_half_and_zero_rhs_bitwise():
    # theta = 0.5: the right-hand operator M - k dt/2 K is non-trivial; a zero
    # right-hand side returns zero without iterating (solvers.hpp:28-32)
    d = E.SpatialDiscretization.build(2, 5)
    dt = 2e-3
    st = E.ThetaStepper(d, 1.0, dt, 0.5, _cfg(True))
    ost = O.OcStepper(O.OcDisc(d.operators()), 1.0, dt, 0.5, kind=1)
    rng = np.random.default_rng(37)
    u = rng.standard_normal((2, d.n_free))
    u[1] = 0.0
    guess = rng.standard_normal((2, d.n_free))
    got = st.step(u, None, guess)
    for i in range(2):
        ref, _ = ost.step(u[i], None, guess[i])
        assert np.array_equal(got[i], ref)
    assert not np.any(got[1])


def test_cg_sequential_integrate_bitwise():
    d = E.SpatialDiscretization.build(2, 4)
    nt, dt = 16, 0.1 / 16
    st = E.ThetaStepper(d, 1.0, dt, 1.0, _cfg(True))
    od = O.OcDisc(d.operators())
    u0 = np.random.default_rng(41).uniform(-1, 1, d.n_free)
    got, solves, its = st.sequential_integrate(nt, u0, None)
    ost = O.OcStepper(od, 1.0, dt, 1.0, kind=1)
    u = u0.copy()
    total = 0
    for k in range(nt):
        u, it = ost.step(u, None, u)
        total += it
        assert np.array_equal(got[k + 1], u)
    assert solves == nt and its == total
