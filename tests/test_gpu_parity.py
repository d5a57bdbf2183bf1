"""GPU parity: the CUDA engine (through its C ABI) against the reference.

Bar: bit-identical.  In its exact mode (phi_pmg_options.exact = 1) the
engine evaluates every reference reduction in the reference's order without
fused multiply-adds, so operators, V-cycles,
solves, Phi steps and MGRIT trajectories must equal the reference (oracle/_ref,
the unmodified reference compiled from /root/reference) and the C restatement
(oracle/phi_oracle.c) exactly.  np.array_equal is the assertion throughout.
"""
import numpy as np
import pytest

from oracle import oracle as O
from tests.conftest import gpu_available

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]

E = pytest.importorskip("paper_2107_05337_b200.engine")
# the bitwise tests run the engine in its exact mode (reference summation
# order); the default reassociated mode is covered by test_gpu_fast.py
EXACT = E.default_solver_config(exact=1)


def _same_csr(a, b, what):
    assert (a.n_rows, a.n_cols) == (b.n_rows, b.n_cols), what
    assert np.array_equal(a.row_offsets, b.row_offsets), what
    assert np.array_equal(a.col_indices, b.col_indices), what
    assert np.array_equal(a.values, b.values), (what, np.max(np.abs(a.values - b.values)))


def _ref_or_skip():
    if not O.ref_available():
        pytest.skip("oracle/_ref not built (make -C oracle ref)")


_disc_cache = {}


def disc(p, k):
    if (p, k) not in _disc_cache:
        _disc_cache[(p, k)] = E.SpatialDiscretization.build(p, k)
    return _disc_cache[(p, k)]


@pytest.mark.parametrize("p,k", [(1, 3), (2, 4), (3, 5), (4, 4), (5, 5), (3, 6)])
def test_device_assembly_matches_reference(p, k):
    _ref_or_skip()
    d = disc(p, k)
    r = O.RefDisc(p, k)
    assert (d.n_free, d.n_h_levels) == (r.n_free, r.n_h)
    for which in [0, 1, 2] + [100 + l for l in range(r.n_h)] + [200 + l for l in range(r.n_h)] \
            + [300 + l for l in range(r.n_h - 1)]:
        _same_csr(d.csr(which), r.csr(which), f"disc {which}")
    assert np.array_equal(d.vec(0), r.vec(0))
    assert np.array_equal(d.vec(1), r.vec(1))


@pytest.mark.parametrize("p,k,c", [(2, 4, 1e-3), (3, 5, 1e-4), (5, 5, 0.01)])
def test_hierarchy_matches_reference(p, k, c):
    _ref_or_skip()
    d = disc(p, k)
    h = E.PMultigridHierarchy(d, c, exact=True)
    r = O.RefHier(O.RefDisc(p, k), c)
    for which in [0, 1, 2] + [100 + l for l in range(d.n_h_levels)]:
        _same_csr(h.csr(which), r.csr(which), f"hier {which}")


def _oc(d: "E.SpatialDiscretization", c):
    od = O.OcDisc(d.operators())
    return od, O.OcHier(od, c)


@pytest.mark.parametrize("p,k,c", [(2, 4, 1e-3), (3, 5, 1e-4), (4, 5, 4e-5)])
def test_building_blocks_bitwise(p, k, c):
    d = disc(p, k)
    h = E.PMultigridHierarchy(d, c, exact=True)
    od, oh = _oc(d, c)
    rng = np.random.default_rng(7)
    r = rng.standard_normal(d.n_free)
    x = rng.standard_normal(d.n_free)
    assert np.array_equal(h.spmv(x), O.oc_spmv(oh.csr(0), x))
    assert np.array_equal(h.ilut_apply(r), oh.ilut_apply(r))
    r1 = h.restrict_to_linear(r)
    assert np.array_equal(r1, oh.restrict(r))
    e1 = rng.standard_normal(d.n_free_1)
    assert np.array_equal(h.prolong_from_linear(e1), oh.prolong(e1))
    assert np.array_equal(h.hmg_wcycle(r1), oh.hmg_wcycle(r1))
    a0 = oh.csr(100)
    b1 = rng.standard_normal(d.n_free_1)
    x1 = rng.standard_normal(d.n_free_1)
    for back in (False, True):
        assert np.array_equal(h.gauss_seidel_sweep(0, b1, x1, back), O.oc_gs_sweep(a0, b1, x1, back))


@pytest.mark.parametrize("p,k,c,nrhs", [(2, 4, 1e-3, 5), (3, 6, 1e-4, 3), (5, 5, 1e-4, 2)])
def test_vcycle_batched_bitwise(p, k, c, nrhs):
    d = disc(p, k)
    h = E.PMultigridHierarchy(d, c, exact=True)
    od, oh = _oc(d, c)
    rng = np.random.default_rng(11)
    b = rng.standard_normal((nrhs, d.n_free))
    x = rng.standard_normal((nrhs, d.n_free))
    got = h.vcycle(b, x)
    for i in range(nrhs):
        assert np.array_equal(got[i], oh.vcycle(b[i], x[i]))


def test_solve_batched_bitwise_with_zero_rhs_and_early_exit():
    d = disc(3, 5)
    c = 1e-3
    h = E.PMultigridHierarchy(d, c, exact=True)
    od, oh = _oc(d, c)
    rng = np.random.default_rng(3)
    b = rng.standard_normal((4, d.n_free))
    b[1] = 0.0  # zero rhs -> x = 0, 0 iterations (pmultigrid.hpp:274-279)
    x0 = rng.standard_normal((4, d.n_free))
    x0[2] = oh.solve(b[2], rel_tol=1e-14, max_iter=50)["x"]  # already converged -> 0 its
    got = h.solve(b, x0, rel_tol=1e-12, max_iter=400)
    for i in range(4):
        ref = oh.solve(b[i], x0[i], rel_tol=1e-12, max_iter=400)
        assert got["iterations"][i] == ref["iterations"]
        assert got["converged"][i] == ref["converged"]
        assert np.array_equal(got["x"][i], ref["x"])
        assert got["final_relative_residual"][i] == ref["final_relative_residual"]
    assert got["iterations"][1] == 0 and not np.any(got["x"][1])


def test_solve_fixed_cycles_and_x0_empty():
    d = disc(2, 5)
    h = E.PMultigridHierarchy(d, 0.01, exact=True)
    od, oh = _oc(d, 0.01)
    b = np.random.default_rng(5).standard_normal(d.n_free)
    got = h.solve(b, None, fixed_cycles=3)
    ref = oh.solve(b, None, fixed_cycles=3)
    assert got["iterations"] == 3 and np.array_equal(got["x"], ref["x"])


@pytest.mark.parametrize("theta", [1.0, 0.5])
def test_theta_step_bitwise(theta):
    d = disc(2, 5)
    dt = 1e-3
    st = E.ThetaStepper(d, 1.0, dt, theta, EXACT)
    od = O.OcDisc(d.operators())
    ost = O.OcStepper(od, 1.0, dt, theta)
    rng = np.random.default_rng(13)
    u = rng.standard_normal((3, d.n_free))
    load = rng.standard_normal((3, d.n_free))
    guess = rng.standard_normal((3, d.n_free))
    got = st.step(u, load, guess)
    for i in range(3):
        ref, _ = ost.step(u[i], load[i], guess[i])
        assert np.array_equal(got[i], ref)


def test_sequential_integrate_bitwise():
    d = disc(2, 4)
    nt, dt = 32, 0.1 / 32
    st = E.ThetaStepper(d, 1.0, dt, 1.0, EXACT)
    od = O.OcDisc(d.operators())
    u0 = np.random.default_rng(17).uniform(-1, 1, d.n_free)
    load = np.full(d.n_free, 1e-3)
    got, solves, its = st.sequential_integrate(nt, u0, load, load_steady=True)
    ref, rs, rit = O.oc_sequential_integrate(od, nt, t_final=0.1, u0=u0, loads=load, load_steady=True)
    assert np.array_equal(got, ref) and (solves, its) == (rs, rit)


def _mgrit_pair(p, k, nt, **kw):
    _ref_or_skip()
    d = disc(p, k)
    eng = E.MgritSolver(d, nt, exact=True, **kw)
    ref = O.RefMgrit(p, k, nt, **kw)
    return eng, ref


@pytest.mark.parametrize("case", [
    # config 1 of BASELINE.json (reference probe: 5 iterations, 2000 solves)
    dict(p=2, k=4, nt=100, m=4, cycle=E.CYCLE_TWO_LEVEL, source_param=0.0, init_kind=E.INIT_SIN),
    # multilevel V and F cycles, steady unit source (the reference's model problem)
    dict(p=2, k=3, nt=64, m=2, cycle=E.CYCLE_V),
    dict(p=3, k=3, nt=32, m=2, cycle=E.CYCLE_F, relax=E.RELAX_F),
    # transient source + spline initial coefficients (config-2 shape, smaller)
    dict(p=3, k=5, nt=64, m=8, cycle=E.CYCLE_TWO_LEVEL, source_kind=E.SOURCE_SIN_EXP,
         source_param=2 * np.pi ** 2, init_kind=E.INIT_COEFFS),
])
def test_mgrit_bitwise_vs_reference(case):
    case = dict(case)
    p, k, nt = case.pop("p"), case.pop("k"), case.pop("nt")
    if case.get("init_kind") == E.INIT_COEFFS:
        n = (2 ** k + p - 2) ** 2
        case["init_coeffs"] = np.random.default_rng(12345).uniform(-1, 1, n)
    eng, ref = _mgrit_pair(p, k, nt, **case)
    assert eng.levels() == ref.levels()
    rg = eng.solve()
    rr = ref.solve()
    assert rg.iterations == rr["iterations"]
    assert rg.converged == rr["converged"]
    assert rg.total_spatial_solves == rr["total_spatial_solves"]
    assert rg.mean_spatial_iterations == rr["mean_spatial_iterations"]
    assert rg.g_norm == rr["g_norm"]
    assert np.array_equal(rg.residual_history, rr["residual_history"])
    assert np.array_equal(eng.trajectory(), ref.trajectory())
