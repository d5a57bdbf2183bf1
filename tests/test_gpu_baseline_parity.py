"""Parity of the BENCHMARKED mode (reassociated sums, exact = 0) against the
reference compiled here (oracle/_ref), at BASELINE.json sizes.

The north-star bar (BASELINE.json): MGRIT and p-multigrid iteration counts
within +-1 and the final space-time solution within 1e-8 relative L2 (fp64).
The reference's own equivalence gates are tests/test_mgrit.cpp:320-335
(MGRIT vs sequential, 1e-8) and acceptance.cpp:74-97 (criterion 1).

p-multigrid counts are compared PER SOLVE: after every MGRIT iteration both
sides run the residual wave of level 0 (one Phi solve per time point,
mgrit.hpp:197-214) on their own state and report each solve's cycle count
(engine: phi_mgrit_residual_iters; reference: ThetaStepper::step per point
with its own SolveStats, oracle/ref_driver.cpp ref_mgrit_residual_iters).
Every solve must agree within +-1.  Totals over the whole solve (solves and
mean cycles per solve) are compared as well.

Cases:
  * config 2 in full (p=3, h=2^-6, Nt=1000, two-level m=8, the bench's inputs);
  * config 3 (p=4, h=2^-7, Nt=2500, m=4): initialize + 2 MGRIT iterations;
  * config-4 shape (p=5, h=2^-8, m=8, transient source, u0 = 0) at Nt=48,
    in both summation modes -- the exact mode bit for bit;
  * one V(1,1) cycle and full solves at h=2^-8 for p = 2..5 (config 5);
  * the multilevel variants: config 3 at Nt=2560 with
    coarse_floor 41 (3 levels 2560/640/160), initialize + 2 iterations, and
    the config-4 operator over 3 levels (Nt=128, m=4: 128/32/8) to
    convergence, both modes.
"""
import os

import numpy as np
import pytest

from oracle import oracle as O
from tests.conftest import gpu_available

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]

E = pytest.importorskip("paper_2107_05337_b200.engine")

TOL_TRAJ = 1e-8  # north star: space-time solution, relative L2
SEED = 12345     # bench.py's seed for the U[-1, 1] initial coefficients
WORKERS = os.cpu_count() or 1


def _rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


def _need_ref():
    if not O.ref_available():
        pytest.skip("oracle/_ref not built (make -C oracle ref)")


def _coeffs(p, k):
    return np.random.default_rng(SEED).uniform(-1.0, 1.0, (2 ** k + p - 2) ** 2)


def _pair(p, k, nt, exact=False, **kw):
    eng = E.MgritSolver(E.SpatialDiscretization.build(p, k), nt, exact=exact, **kw)
    ref = O.RefMgrit(p, k, nt, workers=WORKERS, **kw)
    assert eng.levels()[0] == ref.levels()[0]
    return eng, ref


def _step_and_compare(eng, ref, iters):
    """Both sides: initialize, then `iters` MGRIT iterations (None: to the
    halting tolerance).  After each iteration compare the per-solve p-MG
    counts of the residual wave and the relative residual."""
    g_e, g_r = eng.initialize(), ref.initialize()
    assert abs(g_e - g_r) <= 1e-10 * g_r
    denom = g_r if g_r > 0 else 1.0
    hist_e, hist_r, worst, differ = [], [], 0, 0
    it = 0
    while True:
        it += 1
        eng.mgrit_cycle(0)
        ref.mgrit_cycle(0)
        ie, ir = eng.residual_iters(0), ref.residual_iters(0, WORKERS)
        d = np.abs(ie.astype(int) - ir.astype(int))
        worst = max(worst, int(d.max()))
        differ += int((d > 0).sum())
        assert d.max() <= 1, (it, np.nonzero(d > 1)[0][:10])
        re, rr = eng.residual_norm(0) / denom, ref.residual_norm(0) / denom
        hist_e.append(re)
        hist_r.append(rr)
        if iters is not None and it == iters:
            break
        if iters is None and (rr <= 1e-10 or re <= 1e-10 or it >= 50):
            break
    return np.array(hist_e), np.array(hist_r), worst, differ


@pytest.mark.slow
def test_config2_full_solve_matches_reference():
    """BASELINE config 2 end to end: iterations, per-solve p-MG counts,
    totals and the whole trajectory."""
    _need_ref()
    p, k, nt = 3, 6, 1000
    kw = dict(cycle=E.CYCLE_TWO_LEVEL, m=8, source_kind=E.SOURCE_SIN_EXP, source_param=2 * np.pi ** 2,
              init_kind=E.INIT_COEFFS, init_coeffs=_coeffs(p, k))
    eng, ref = _pair(p, k, nt, **kw)
    he, hr, worst, differ = _step_and_compare(eng, ref, None)
    assert len(he) == len(hr), (he, hr)  # same MGRIT iteration count (8 at C2)
    assert he[-1] <= 1e-10 and hr[-1] <= 1e-10
    # the residual history agrees far below the halting tolerance
    assert np.all(np.abs(he - hr) <= 1e-3 * hr + 1e-13)
    # whole solve(): counts and trajectory
    re_, rr = eng.solve(), ref.solve()
    assert re_.iterations == rr["iterations"]
    assert re_.total_spatial_solves == rr["total_spatial_solves"]
    assert abs(re_.mean_spatial_iterations - rr["mean_spatial_iterations"]) <= 0.01
    assert _rel(eng.trajectory(), ref.trajectory()) <= TOL_TRAJ
    print(f"C2: {len(he)} iterations, per-solve p-MG differences {differ} (max {worst}), "
          f"mean {re_.mean_spatial_iterations:.4f} vs {rr['mean_spatial_iterations']:.4f}")


@pytest.mark.slow
def test_config3_two_iterations_match_reference():
    """BASELINE config 3 (p=4, h=2^-7, Nt=2500, m=4, seeded u0, f=0):
    initialize + 2 MGRIT iterations, per-solve counts and the state."""
    _need_ref()
    p, k, nt = 4, 7, 2500
    kw = dict(cycle=E.CYCLE_V, m=4, source_param=0.0, init_kind=E.INIT_COEFFS, init_coeffs=_coeffs(p, k))
    eng, ref = _pair(p, k, nt, **kw)
    assert eng.levels()[0] == [2500, 625]  # the reference builds two levels here
    he, hr, worst, differ = _step_and_compare(eng, ref, 2)
    assert np.all(np.abs(he - hr) <= 1e-6 * hr)
    ue = np.empty((nt + 1, eng.disc.n_free))
    for k0 in range(0, nt + 1, 500):
        c = min(500, nt + 1 - k0)
        ue[k0:k0 + c] = ref.points(0, 0, k0, c)
    assert _rel(eng.trajectory(), ue) <= TOL_TRAJ
    print(f"C3: 2 iterations, residual {he[-1]:.3e} vs {hr[-1]:.3e}, per-solve differences {differ}")


@pytest.fixture(scope="module")
def c4_shape():
    """Config-4 operator (p=5, h=2^-8), m=8, transient 2 pi^2 e^-t sin sin
    source, u0 = 0, at Nt=48 (levels 48 / 6): the reference run once."""
    _need_ref()
    p, k, nt = 5, 8, 48
    kw = dict(cycle=E.CYCLE_V, m=8, source_kind=E.SOURCE_SIN_EXP, source_param=2 * np.pi ** 2)
    ref = O.RefMgrit(p, k, nt, workers=WORKERS, **kw)
    rr = ref.solve()
    return dict(p=p, k=k, nt=nt, kw=kw, ref=ref, res=rr, traj=ref.trajectory())


@pytest.mark.slow
def test_config4_shape_exact_mode_bitwise(c4_shape):
    """Exact mode at h=2^-8, p=5: bit-identical to the reference."""
    c = c4_shape
    eng = E.MgritSolver(E.SpatialDiscretization.build(c["p"], c["k"]), c["nt"], exact=True, **c["kw"])
    r = eng.solve()
    assert r.iterations == c["res"]["iterations"]
    assert r.total_spatial_solves == c["res"]["total_spatial_solves"]
    assert r.mean_spatial_iterations == c["res"]["mean_spatial_iterations"]
    assert np.array_equal(r.residual_history, c["res"]["residual_history"])
    assert np.array_equal(eng.trajectory(), c["traj"])


@pytest.mark.slow
def test_config4_shape_fast_mode_per_solve(c4_shape):
    """Benchmarked mode at h=2^-8, p=5: per-solve p-MG counts, iterations,
    totals and the trajectory."""
    c = c4_shape
    eng = E.MgritSolver(E.SpatialDiscretization.build(c["p"], c["k"]), c["nt"], **c["kw"])
    ref = c["ref"]
    he, hr, worst, differ = _step_and_compare(eng, ref, c["res"]["iterations"])
    assert hr[-1] == pytest.approx(c["res"]["final_relative_residual"], rel=1e-12)
    r = eng.solve()
    assert abs(r.iterations - c["res"]["iterations"]) <= 1
    assert r.converged
    assert r.total_spatial_solves == c["res"]["total_spatial_solves"]
    assert abs(r.mean_spatial_iterations - c["res"]["mean_spatial_iterations"]) <= 0.02
    assert _rel(eng.trajectory(), c["traj"]) <= TOL_TRAJ


@pytest.mark.slow
@pytest.mark.parametrize("p", [2, 3, 4, 5])
def test_config5_vcycle_and_solve_k8(p):
    """Config 5 shapes (h=2^-8, c=1e-4): one V(1,1) on seeded N(0,1)
    right-hand sides from x0 = 0, and full solves with per-solve counts."""
    _need_ref()
    k, c = 8, 1e-4
    d = E.SpatialDiscretization.build(p, k)
    h = E.PMultigridHierarchy(d, c)
    r = O.RefHier(O.RefDisc(p, k), c)
    rng = np.random.default_rng(100 + p)
    B = rng.standard_normal((3, d.n_free))
    X = h.vcycle(B, np.zeros_like(B))
    for i in range(3):
        assert _rel(X[i], r.vcycle(B[i], np.zeros(d.n_free))) <= 1e-10
    got = h.solve(B, None)
    for i in range(3):
        ref = r.solve(B[i])
        assert abs(int(got["iterations"][i]) - ref["iterations"]) <= 1
        assert got["converged"][i]
        assert _rel(got["x"][i], ref["x"]) <= 1e-9


@pytest.mark.slow
def test_config3_multilevel_variant_two_iterations():
    """C3 operator, Nt=2560, m=4, coarse_floor=41: the reference's three
    levels 2560/640/160 (bench.py --config c3ml)."""
    _need_ref()
    p, k, nt = 4, 7, 2560
    kw = dict(cycle=E.CYCLE_V, m=4, source_param=0.0, init_kind=E.INIT_COEFFS, init_coeffs=_coeffs(p, k),
              coarse_floor=41)
    eng, ref = _pair(p, k, nt, **kw)
    assert eng.levels()[0] == [2560, 640, 160]
    he, hr, worst, differ = _step_and_compare(eng, ref, 2)
    assert np.all(np.abs(he - hr) <= 1e-6 * hr)
    ur = np.concatenate([ref.points(0, 0, k0, min(512, nt + 1 - k0)) for k0 in range(0, nt + 1, 512)])
    assert _rel(eng.trajectory(), ur) <= TOL_TRAJ


@pytest.fixture(scope="module")
def c4_multilevel():
    """C4 operator and source over three levels (Nt=128, m=4: 128/32/8)."""
    _need_ref()
    p, k, nt = 5, 8, 128
    kw = dict(cycle=E.CYCLE_V, m=4, source_kind=E.SOURCE_SIN_EXP, source_param=2 * np.pi ** 2)
    ref = O.RefMgrit(p, k, nt, workers=WORKERS, **kw)
    assert ref.levels()[0] == [128, 32, 8]
    rr = ref.solve()
    return dict(p=p, k=k, nt=nt, kw=kw, ref=ref, res=rr, traj=ref.trajectory())


@pytest.mark.slow
@pytest.mark.parametrize("exact", [True, False])
def test_config4_multilevel_shape(c4_multilevel, exact):
    c = c4_multilevel
    eng = E.MgritSolver(E.SpatialDiscretization.build(c["p"], c["k"]), c["nt"], exact=exact, **c["kw"])
    r = eng.solve()
    if exact:
        assert r.iterations == c["res"]["iterations"]
        assert r.total_spatial_solves == c["res"]["total_spatial_solves"]
        assert np.array_equal(r.residual_history, c["res"]["residual_history"])
        assert np.array_equal(eng.trajectory(), c["traj"])
    else:
        assert abs(r.iterations - c["res"]["iterations"]) <= 1 and r.converged
        assert r.total_spatial_solves == c["res"]["total_spatial_solves"]
        assert abs(r.mean_spatial_iterations - c["res"]["mean_spatial_iterations"]) <= 0.02
        assert _rel(eng.trajectory(), c["traj"]) <= TOL_TRAJ


@pytest.mark.parametrize("exact", [True, False])
def test_fcycle_four_levels_golden(exact):
    """F-cycle over four levels against the committed reference fixture
    (tests/golden/mgrit_fcycle.npz): bitwise in exact mode."""
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "mgrit_fcycle.npz"))
    p, k, nt = 2, 3, 64
    eng = E.MgritSolver(E.SpatialDiscretization.build(p, k), nt, cycle=E.CYCLE_F, m=2,
                        source_kind=E.SOURCE_SIN_EXP, source_param=2 * np.pi ** 2, init_kind=E.INIT_COEFFS,
                        init_coeffs=g["coeffs"], exact=exact)
    assert eng.levels()[0] == [int(v) for v in g["levels_steps"]]
    r = eng.solve()
    if exact:
        assert r.iterations == int(g["iterations"][0])
        assert r.total_spatial_solves == int(g["solves"][0])
        assert np.array_equal(r.residual_history, g["history"])
        assert np.array_equal(eng.trajectory(), g["trajectory"])
    else:
        assert abs(r.iterations - int(g["iterations"][0])) <= 1
        assert _rel(eng.trajectory(), g["trajectory"]) <= TOL_TRAJ


@pytest.mark.parametrize("p,k", [(3, 6), (4, 7)])
def test_initial_projection_on_a_cluster_matches_reference(p, k):
    """project_initial (theta.hpp:150-210: Jacobi CG on M, solvers.hpp:21-75) at the sizes
    of configs 2 and 3, where the device CG runs on a cluster of CTAs (n >= 4096): the
    projected u0 is bitwise the reference's in exact mode (rows split over the cluster,
    whole-vector dot products in every CTA) and within the trajectory bar in the default
    mode; both repeatable bit for bit."""
    _need_ref()
    kw = dict(cycle=E.CYCLE_TWO_LEVEL, m=4, init_kind=E.INIT_COEFFS, init_coeffs=_coeffs(p, k), source_param=0.0)
    ref = O.RefMgrit(p, k, 8, workers=WORKERS, **kw)
    ref.initialize()
    u_ref = ref.initial()
    disc = E.SpatialDiscretization.build(p, k)
    for exact in (True, False):
        got = []
        for _ in range(2):
            eng = E.MgritSolver(disc, 8, exact=exact, **kw)
            eng.initialize()
            got.append(eng.initial())
        assert np.array_equal(got[0], got[1])
        if exact:
            assert np.array_equal(got[0], u_ref)
        else:
            assert _rel(got[0], u_ref) <= 1e-12
