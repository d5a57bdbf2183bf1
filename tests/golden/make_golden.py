"""Generate the golden fixtures of tests/golden/ from the compiled reference.

TEST INFRASTRUCTURE.  Runs the UNMODIFIED reference (`miga`, header-only C++,
compiled by `make -C oracle ref` into oracle/_ref/libmiga_ref.so from its own
headers under /root/reference) on small seeded inputs and stores what it
returns.  The GPU box has no /root/reference, so the CPU tests pin the oracle's
C restatement against these files, and the GPU tests can use them where the
compiled reference is absent.

    python tests/golden/make_golden.py        # rewrites tests/golden/*.npz

Fixtures
  ops_p2k3.npz    SpatialDiscretization::build(2, 3) arrays (pmultigrid.hpp:94-158),
                  PMultigridHierarchy(disc, 1e-3) factors L/U and a_h (pmultigrid.hpp:215-240),
                  and the building blocks on seeded vectors: ilut_apply (ilut.hpp:146-163),
                  restrict/prolong (pmultigrid.hpp:242-254), hmg_wcycle (172-200),
                  gauss_seidel_sweep fwd/bwd (solvers.hpp:80-99), the 9x9 coarse LU
                  (solvers.hpp:102-172), vcycle (256-267) and solve (271-307).
  setup_host.npz  the reference's host setup on the shapes of BASELINE.json configs 1-5:
                  detail::DirTables (assembly.hpp:124-151: gauss_legendre_01, open_uniform_knots,
                  eval_values_and_derivs) for (degree, elements, points) of the degree-p and the
                  order-1 spaces, and DenseLU(a).solve(b) (solvers.hpp:102-172) on seeded dense
                  systems (full, sparse with a zero diagonal that forces pivoting) with their inputs.
  mgrit_*.npz     also hold the SpatialDiscretization arrays of their (p, h).
  mgrit_c1.npz    BASELINE.json config 1 (p=2, h=2^-4, Nt=100, two-level m=4, FCF,
                  f=0, u0=sin sin): MgritSolver::solve() (mgrit.hpp:93-118) result,
                  residual history, projected u0 and the trajectory.
  mgrit_cg.npz    as mgrit_src.npz with the CG spatial solver (theta.hpp:121-125)
  mgrit_fcycle.npz  F-cycle (cycle=F, FCF) over 4 levels (p=2, h=2^-3, Nt=64, m=2:
                  64/32/16/8), transient source, spline u0: the F-schedule's second
                  pass (mgrit.hpp:278-288) with a coarse cycle below it.
  mgrit_src.npz   the config-2 shape at small size (p=3, h=2^-4, Nt=32, m=8, transient
                  2 pi^2 e^-t sin sin source, spline u0 from seeded U[-1,1] coefficients):
                  result, u0, the level-0 load terms and the trajectory.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402


def _csr(prefix: str, a: O.CSR, out: dict) -> None:
    out[prefix + "_shape"] = np.array([a.n_rows, a.n_cols], np.int32)
    out[prefix + "_ro"] = np.asarray(a.row_offsets, np.int32)
    out[prefix + "_ci"] = np.asarray(a.col_indices, np.int32)
    out[prefix + "_v"] = np.asarray(a.values, np.float64)


def _store_ops(ops: dict, out: dict) -> None:
    for key in ("mass_p", "stiff_p", "transfer"):
        _csr(key, ops[key], out)
    out["inv_lumped_p"] = ops["inv_lumped_p"]
    out["inv_lumped_1"] = ops["inv_lumped_1"]
    out["n_h"] = np.array([len(ops["h_mass"])], np.int32)
    for l, a in enumerate(ops["h_mass"]):
        _csr(f"h_mass{l}", a, out)
    for l, a in enumerate(ops["h_stiff"]):
        _csr(f"h_stiff{l}", a, out)
    for l, a in enumerate(ops["h_embed"]):
        _csr(f"h_embed{l}", a, out)


def ops_fixture() -> dict:
    out: dict = {}
    d = O.RefDisc(2, 3)
    ops = d.operators()
    _store_ops(ops, out)
    c = 1e-3
    out["c"] = np.array([c])
    h = O.RefHier(d, c)
    _csr("A", h.csr(0), out)
    _csr("L", h.csr(1), out)
    _csr("U", h.csr(2), out)
    for l in range(len(ops["h_mass"])):
        _csr(f"a_h{l}", h.csr(100 + l), out)
    n, n1 = ops["mass_p"].n_rows, ops["transfer"].n_cols
    rng = np.random.default_rng(20240611)
    b = rng.uniform(-1.0, 1.0, n)
    b1 = rng.uniform(-1.0, 1.0, n1)
    x1 = rng.uniform(-1.0, 1.0, n1)
    out["b"], out["b1"], out["x1"] = b, b1, x1
    out["ilut_apply"] = h.ilut_apply(b)
    out["restrict"] = h.restrict(b)
    out["prolong"] = h.prolong(b1)
    out["wcycle"] = h.hmg_wcycle(b1)
    out["gs_fwd"] = h.gs_sweep(0, b1, x1, backward=False)
    out["gs_bwd"] = h.gs_sweep(0, b1, x1, backward=True)
    nc = ops["h_mass"][-1].n_rows
    out["bc"] = b1[:nc].copy()
    out["coarse"] = h.coarse_solve(out["bc"])
    out["vcycle"] = h.vcycle(b, np.zeros(n))
    s = h.solve(b)
    out["solve_x"], out["solve_iters"] = s["x"], np.array([s["iterations"]], np.int32)
    out["solve_hist"] = s["residual_history"]
    return out


def mgrit_fixture(p, k, nt, **kw) -> dict:
    g = O.RefMgrit(p, k, nt, **kw)
    steps, dts = g.levels()
    r = g.solve()
    out = {"levels_steps": np.array(steps, np.int32), "levels_dts": np.array(dts),
           "iterations": np.array([r["iterations"]], np.int32),
           "converged": np.array([int(r["converged"])], np.int32),
           "g_norm": np.array([r["g_norm"]]), "final_rel": np.array([r["final_relative_residual"]]),
           "solves": np.array([r["total_spatial_solves"]], np.int64),
           "mean_iters": np.array([r["mean_spatial_iterations"]]),
           "history": r["residual_history"], "u0": g.initial(), "trajectory": g.trajectory()}
    _store_ops(O.RefDisc(p, k).operators(), out)
    loads = g.load_terms()
    if loads is not None:
        out["loads"] = loads
    return out


# (degree, elements, points per span): degree-p spaces of configs 1-5 at small and BASELINE
# mesh sizes with their p+1 rule, and the order-1 spaces (2-point rule, and sampled at the
# degree-p nodes through a (p+1)-point rule)
SETUP_TABLE_CASES = [(2, 16, 3), (3, 64, 4), (4, 128, 5), (5, 256, 6), (2, 256, 3), (3, 256, 4),
                     (1, 256, 2), (1, 128, 2), (1, 2, 2), (1, 16, 3), (1, 64, 6), (2, 1, 3), (5, 3, 6)]
SETUP_LU_SIZES = [1, 2, 9, 25, 49]


def setup_lu_inputs():
    """Seeded dense systems: a full one, and one with a zero diagonal (pivoting) per size."""
    rng = np.random.default_rng(777)
    out = []
    for n in SETUP_LU_SIZES:
        full = rng.uniform(-1.0, 1.0, (n, n))
        holed = np.where(rng.uniform(size=(n, n)) < 0.5, rng.uniform(-1.0, 1.0, (n, n)), 0.0)
        np.fill_diagonal(holed, 0.0)
        holed += 0.75 * np.roll(np.eye(n), 1, axis=1) if n > 1 else 1.0
        out.append((full, rng.standard_normal(n)))
        out.append((holed, rng.standard_normal(n)))
    return out


def setup_fixture() -> dict:
    out: dict = {}
    for (p, nel, nq) in SETUP_TABLE_CASES:
        for k, v in O.ref_tables_1d(p, nel, nq).items():
            out[f"t_{p}_{nel}_{nq}_{k}"] = v
    for i, (a, b) in enumerate(setup_lu_inputs()):
        out[f"lu{i}_a"], out[f"lu{i}_b"] = a, b
        out[f"lu{i}_x"] = O.ref_dense_solve(a, b)
    return out


def fixtures() -> dict:
    """name -> builder of each committed fixture."""
    coeffs = np.random.default_rng(12345).uniform(-1.0, 1.0, (2 ** 4 + 3 - 2) ** 2)
    coeffs3 = np.random.default_rng(12345).uniform(-1.0, 1.0, (2 ** 3 + 2 - 2) ** 2)
    return {
        "ops_p2k3.npz": ops_fixture,
        "setup_host.npz": setup_fixture,
        "mgrit_c1.npz": lambda: mgrit_fixture(2, 4, 100, cycle=O.CYCLE_TWO_LEVEL, m=4,
                                              source_param=0.0, init_kind=O.INIT_SIN),
        "mgrit_src.npz": lambda: dict(coeffs=coeffs, **mgrit_fixture(
            3, 4, 32, cycle=O.CYCLE_TWO_LEVEL, m=8, source_kind=O.SOURCE_SIN_EXP,
            source_param=2 * np.pi ** 2, init_kind=O.INIT_COEFFS, init_coeffs=coeffs)),
        "mgrit_fcycle.npz": lambda: dict(coeffs=coeffs3, **mgrit_fixture(
            2, 3, 64, cycle=O.CYCLE_F, m=2, source_kind=O.SOURCE_SIN_EXP, source_param=2 * np.pi ** 2,
            init_kind=O.INIT_COEFFS, init_coeffs=coeffs3)),
        # the CG spatial-solver kind (SpatialSolverKind::cg, theta.hpp:64, 121-125)
        "mgrit_cg.npz": lambda: dict(coeffs=coeffs, **mgrit_fixture(
            3, 4, 32, cycle=O.CYCLE_TWO_LEVEL, m=8, source_kind=O.SOURCE_SIN_EXP,
            source_param=2 * np.pi ** 2, init_kind=O.INIT_COEFFS, init_coeffs=coeffs,
            spatial_kind=1)),
    }


def main(only=None) -> None:
    if not O.ref_available():
        raise SystemExit("oracle/_ref missing: run `make -C oracle ref` (needs /root/reference)")
    for name, make in fixtures().items():
        if only and name not in only:
            continue
        np.savez_compressed(os.path.join(HERE, name), **make())
    for f in sorted(os.listdir(HERE)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(HERE, f)), "bytes")


if __name__ == "__main__":
    import sys

    main(sys.argv[1:] or None)
