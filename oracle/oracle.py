"""TEST INFRASTRUCTURE ONLY -- ctypes bindings for the parity checkers.

* ``Ref*`` classes drive ``oracle/_ref/libmiga_ref.so``: the UNMODIFIED
  reference library (``/root/reference/proj/include/miga``) compiled by
  ``oracle/Makefile`` through ``oracle/ref_driver.cpp``.
* ``Oc*`` classes drive ``oracle/_build/libphi_oracle.so``: the plain-C
  restatement in ``oracle/phi_oracle.c``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs may
import this module.  The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libmiga_ref.so")
OC_SO = os.path.join(HERE, "_build", "libphi_oracle.so")

_vp = C.c_void_p
_i = C.c_int
_d = C.c_double
_ll = C.c_longlong


def _p(a):
    return None if a is None else a.ctypes.data_as(_vp)


@dataclass
class CSR:
    """Mirror of miga::SparseMatrix (sparse.hpp:17-22)."""

    n_rows: int
    n_cols: int
    row_offsets: np.ndarray  # int32, n_rows + 1
    col_indices: np.ndarray  # int32, nnz
    values: np.ndarray  # float64, nnz

    @property
    def nnz(self) -> int:
        return int(self.col_indices.size)

    def dense(self) -> np.ndarray:
        d = np.zeros((self.n_rows, self.n_cols))
        for i in range(self.n_rows):
            s, e = self.row_offsets[i], self.row_offsets[i + 1]
            d[i, self.col_indices[s:e]] = self.values[s:e]
        return d

    def spmv(self, x: np.ndarray) -> np.ndarray:
        """Sequential row-order y = A x in numpy (small cases only)."""
        y = np.zeros(self.n_rows)
        for i in range(self.n_rows):
            s = 0.0
            for e in range(self.row_offsets[i], self.row_offsets[i + 1]):
                s += self.values[e] * x[self.col_indices[e]]
            y[i] = s
        return y


def _fetch_csr(fn, handle, which) -> CSR:
    nr, nc, nnz = _i(), _i(), _i()
    rc = fn(handle, which, C.byref(nr), C.byref(nc), C.byref(nnz), None, None, None)
    if rc:
        raise ValueError(f"csr selector {which} not available")
    ro = np.zeros(nr.value + 1, np.int32)
    ci = np.zeros(nnz.value, np.int32)
    v = np.zeros(nnz.value, np.float64)
    fn(handle, which, None, None, None, _p(ro), _p(ci), _p(v))
    return CSR(nr.value, nc.value, ro, ci, v)


# ---------------------------------------------------------------------------
# reference (compiled from /root/reference)
# ---------------------------------------------------------------------------
_ref = None


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref_lib():
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            raise RuntimeError(f"{REF_SO} missing: build it with `make -C oracle ref`")
        L = C.CDLL(REF_SO)
        L.ref_last_error.restype = C.c_char_p
        L.ref_disc_build.restype = _vp
        L.ref_disc_build.argtypes = [_i, _i, _i]
        L.ref_disc_free.argtypes = [_vp]
        L.ref_disc_info.argtypes = [_vp, _vp]
        L.ref_disc_csr.argtypes = [_vp, _i, _vp, _vp, _vp, _vp, _vp, _vp]
        L.ref_disc_vec.argtypes = [_vp, _i, _vp]
        L.ref_hier_build.restype = _vp
        L.ref_hier_build.argtypes = [_vp, _d, _i, _i, _i, _i, _d, _i]
        L.ref_hier_free.argtypes = [_vp]
        L.ref_hier_csr.argtypes = [_vp, _i, _vp, _vp, _vp, _vp, _vp, _vp]
        L.ref_hier_vcycle.argtypes = [_vp, _vp, _vp, _i, _i]
        L.ref_hier_vcycle_timed.argtypes = [_vp, _vp, _vp, _i, _i, _i]
        L.ref_hier_vcycle_timed.restype = _d
        L.ref_hier_solve.argtypes = [_vp, _vp, _vp, _i, _d, _i, _i, _i, _vp, _vp, _vp, _vp, _i]
        for f in ("ref_ilut_apply", "ref_restrict", "ref_hmg_wcycle", "ref_coarse_solve"):
            getattr(L, f).argtypes = [_vp, _vp, _vp, _i]
        L.ref_prolong.argtypes = [_vp, _vp, _i, _vp]
        L.ref_gs_sweep.argtypes = [_vp, _i, _vp, _vp, _i, _i]
        L.ref_mgrit_create.restype = _vp
        L.ref_mgrit_create.argtypes = [_i, _i, _d, _d, _i, _d, _i, _d, _i, _vp, _i, _i, _i, _d,
                                       _i, _i, _i, _d, _i]
        L.ref_mgrit_create_kind.restype = _vp
        L.ref_mgrit_create_kind.argtypes = [_i, _i, _d, _d, _i, _d, _i, _d, _i, _vp, _i, _i, _i,
                                            _d, _i, _i, _i, _i, _d, _i]
        L.ref_mgrit_free.argtypes = [_vp]
        L.ref_mgrit_levels.argtypes = [_vp, _vp, _vp]
        L.ref_mgrit_solve.argtypes = [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i, _vp]
        L.ref_mgrit_trajectory.argtypes = [_vp, _vp]
        L.ref_mgrit_partial.argtypes = [_vp, _i, _vp, _vp, _vp]
        L.ref_mgrit_initial.argtypes = [_vp, _vp]
        L.ref_load_terms.argtypes = [_vp, _vp]
        L.ref_sequential_integrate.argtypes = [_vp, _vp, _vp, _vp]
        L.ref_mgrit_initialize.argtypes = [_vp, _vp]
        L.ref_mgrit_cycle.argtypes = [_vp, _i]
        L.ref_mgrit_residual_norm.argtypes = [_vp, _i, _vp]
        L.ref_mgrit_points.argtypes = [_vp, _i, _i, _i, _i, _vp]
        L.ref_tables_1d.argtypes = [_i, _i, _i, _vp, _vp, _vp, _vp, _vp]
        L.ref_dense_solve.argtypes = [_i, _vp, _vp, _vp]
        L.ref_mgrit_residual_iters.argtypes = [_vp, _i, _i, _vp]
        _ref = L
    return _ref


def _ref_err():
    return ref_lib().ref_last_error().decode()



def ref_tables_1d(degree: int, n_elements: int, nq: int) -> dict:
    """detail::DirTables of an open uniform knot vector on [0, 1] (assembly.hpp:124-151)."""
    pts = n_elements * nq
    out = dict(nodes=np.empty(pts), weights=np.empty(pts), vals=np.empty((pts, degree + 1)),
               ders=np.empty((pts, degree + 1)), first=np.empty(n_elements, dtype=np.int32))
    L = ref_lib()
    if L.ref_tables_1d(degree, n_elements, nq, _p(out["nodes"]), _p(out["weights"]), _p(out["vals"]),
                       _p(out["ders"]), _p(out["first"])):
        raise ValueError(L.ref_last_error().decode())
    return out


def ref_dense_solve(a, b) -> np.ndarray:
    """DenseLU(a).solve(b) (solvers.hpp:102-172)."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    x = np.empty_like(b)
    L = ref_lib()
    if L.ref_dense_solve(a.shape[0], _p(a), _p(b), _p(x)):
        raise RuntimeError(L.ref_last_error().decode())
    return x


def lu_substitute(lu, piv, b) -> np.ndarray:
    """Permute, forward- and back-substitute with packed LU factors in the order
    of DenseLU::solve (solvers.hpp:118-133); plain Python floats (no fusing)."""
    n = len(piv)
    x = [float(b[int(piv[i])]) for i in range(n)]
    for i in range(n):
        s = x[i]
        for j in range(i):
            s -= float(lu[i][j]) * x[j]
        x[i] = s
    for i in range(n - 1, -1, -1):
        s = x[i]
        for j in range(i + 1, n):
            s -= float(lu[i][j]) * x[j]
        x[i] = s / float(lu[i][i])
    return np.array(x)

class RefDisc:
    """miga::SpatialDiscretization::build on the unit square (pmultigrid.hpp:94-158)."""

    def __init__(self, degree: int, mesh_exponent: int, workers: int = 1):
        L = ref_lib()
        self.h = L.ref_disc_build(degree, mesh_exponent, workers)
        if not self.h:
            raise RuntimeError(_ref_err())
        info = np.zeros(4, np.int32)
        L.ref_disc_info(self.h, _p(info))
        self.n_free, self.n_h, self.n_elements, self.degree = (int(v) for v in info)

    def __del__(self):
        if getattr(self, "h", None):
            ref_lib().ref_disc_free(self.h)

    def csr(self, which: int) -> CSR:
        return _fetch_csr(ref_lib().ref_disc_csr, self.h, which)

    def vec(self, which: int) -> np.ndarray:
        n = self.n_free if which == 0 else self.csr(2).n_cols
        out = np.zeros(n)
        ref_lib().ref_disc_vec(self.h, which, _p(out))
        return out

    def operators(self) -> dict:
        """All SpatialDiscretization arrays the hot path consumes."""
        return {
            "mass_p": self.csr(0),
            "stiff_p": self.csr(1),
            "transfer": self.csr(2),
            "inv_lumped_p": self.vec(0),
            "inv_lumped_1": self.vec(1),
            "h_mass": [self.csr(100 + l) for l in range(self.n_h)],
            "h_stiff": [self.csr(200 + l) for l in range(self.n_h)],
            "h_embed": [self.csr(300 + l) for l in range(self.n_h - 1)],
        }


class RefHier:
    """miga::PMultigridHierarchy (pmultigrid.hpp:215-324)."""

    def __init__(self, disc: RefDisc, c: float, nu_pre=1, nu_post=1, gs_pre=2, gs_post=2,
                 tau=1e-13, fill=0):
        L = ref_lib()
        self.disc = disc
        self.n = disc.n_free
        self.h = L.ref_hier_build(disc.h, c, nu_pre, nu_post, gs_pre, gs_post, tau, fill)
        if not self.h:
            raise RuntimeError(_ref_err())

    def __del__(self):
        if getattr(self, "h", None):
            ref_lib().ref_hier_free(self.h)

    def csr(self, which: int) -> CSR:
        return _fetch_csr(ref_lib().ref_hier_csr, self.h, which)

    def vcycle(self, b: np.ndarray, x: np.ndarray) -> np.ndarray:
        b = np.ascontiguousarray(b, np.float64)
        x = np.array(x, np.float64, copy=True, order="C")
        nrhs = 1 if b.ndim == 1 else b.shape[0]
        if ref_lib().ref_hier_vcycle(self.h, _p(b), _p(x), self.n, nrhs):
            raise RuntimeError(_ref_err())
        return x

    def vcycle_timed(self, b: np.ndarray, x: np.ndarray, workers: int) -> tuple[np.ndarray, float]:
        b = np.ascontiguousarray(b, np.float64)
        x = np.array(x, np.float64, copy=True, order="C")
        t = ref_lib().ref_hier_vcycle_timed(self.h, _p(b), _p(x), self.n, b.shape[0], workers)
        return x, t

    def solve(self, b, x0=None, rel_tol=1e-12, max_iter=400, fixed_cycles=0):
        b = np.ascontiguousarray(b, np.float64)
        x = np.zeros(self.n) if x0 is None else np.array(x0, np.float64, copy=True)
        it, conv, fr = _i(), _i(), _d()
        hist = np.zeros(max(max_iter, fixed_cycles, 1))
        if ref_lib().ref_hier_solve(self.h, _p(b), _p(x), self.n, rel_tol, max_iter, fixed_cycles,
                                    int(x0 is None), C.byref(it), C.byref(conv), C.byref(fr),
                                    _p(hist), hist.size):
            raise RuntimeError(_ref_err())
        return {"x": x, "iterations": it.value, "converged": bool(conv.value),
                "final_relative_residual": fr.value, "residual_history": hist[: it.value].copy()}

    def _unary(self, fn, v, n_out):
        v = np.ascontiguousarray(v, np.float64)
        out = np.zeros(n_out)
        getattr(ref_lib(), fn)(self.h, _p(v), _p(out), v.size)
        return out

    def ilut_apply(self, r):
        return self._unary("ref_ilut_apply", r, self.n)

    def restrict(self, r):
        return self._unary("ref_restrict", r, self.disc.csr(2).n_cols)

    def hmg_wcycle(self, b1, x1=None):
        x = np.zeros(len(b1)) if x1 is None else np.array(x1, np.float64, copy=True)
        ref_lib().ref_hmg_wcycle(self.h, _p(np.ascontiguousarray(b1, np.float64)), _p(x), len(b1))
        return x

    def prolong(self, e1):
        e1 = np.ascontiguousarray(e1, np.float64)
        out = np.zeros(self.n)
        ref_lib().ref_prolong(self.h, _p(e1), e1.size, _p(out))
        return out

    def gs_sweep(self, level, b, x, backward=False):
        x = np.array(x, np.float64, copy=True)
        ref_lib().ref_gs_sweep(self.h, level, _p(np.ascontiguousarray(b, np.float64)), _p(x),
                               x.size, int(backward))
        return x

    def coarse_solve(self, b):
        return self._unary("ref_coarse_solve", b, len(b))


# source / initial kinds shared with include/phi_engine.h
SOURCE_CONSTANT, SOURCE_SIN_EXP, SOURCE_SIN_STEADY = 0, 1, 2
INIT_ZERO, INIT_SIN, INIT_COEFFS = 0, 1, 2
CYCLE_V, CYCLE_F, CYCLE_TWO_LEVEL = 0, 1, 2
RELAX_F, RELAX_FCF = 0, 1


class RefMgrit:
    """miga::MgritSolver over SpatialDiscretization::build (mgrit.hpp:50-331)."""

    def __init__(self, degree, mesh_exponent, nt, *, kappa=1.0, t_final=0.1, theta=1.0,
                 source_kind=SOURCE_CONSTANT, source_param=1.0, init_kind=INIT_ZERO,
                 init_coeffs=None, cycle=CYCLE_V, relax=RELAX_FCF, m=2, halt_tol=1e-10,
                 max_iter=50, coarse_floor=8, workers=1, rel_tol=1e-12, sp_max_iter=400,
                 spatial_kind=0):
        L = ref_lib()
        self._coeffs = None if init_coeffs is None else np.ascontiguousarray(init_coeffs, np.float64)
        self.h = L.ref_mgrit_create_kind(degree, mesh_exponent, kappa, t_final, nt, theta,
                                         source_kind, source_param, init_kind, _p(self._coeffs),
                                         cycle, relax, m, halt_tol, max_iter, coarse_floor, workers,
                                         spatial_kind, rel_tol, sp_max_iter)
        if not self.h:
            raise RuntimeError(_ref_err())
        self.nt = nt
        self.max_iter = max_iter
        self.n = (2 ** mesh_exponent + degree - 2) ** 2

    def __del__(self):
        if getattr(self, "h", None):
            ref_lib().ref_mgrit_free(self.h)

    def levels(self):
        steps = np.zeros(32, np.int32)
        dts = np.zeros(32)
        L = ref_lib().ref_mgrit_levels(self.h, _p(steps), _p(dts))
        return [int(s) for s in steps[:L]], [float(d) for d in dts[:L]]

    def solve(self):
        it, conv, gn, fr, solves, mi, wall = _i(), _i(), _d(), _d(), _ll(), _d(), _d()
        hist = np.zeros(self.max_iter)
        if ref_lib().ref_mgrit_solve(self.h, C.byref(it), C.byref(conv), C.byref(gn), C.byref(fr),
                                     C.byref(solves), C.byref(mi), _p(hist), hist.size,
                                     C.byref(wall)):
            raise RuntimeError(_ref_err())
        return {"iterations": it.value, "converged": bool(conv.value), "g_norm": gn.value,
                "final_relative_residual": fr.value, "total_spatial_solves": solves.value,
                "mean_spatial_iterations": mi.value, "residual_history": hist[: it.value].copy(),
                "wall": wall.value}

    def trajectory(self):
        out = np.zeros((self.nt + 1, self.n))
        ref_lib().ref_mgrit_trajectory(self.h, _p(out))
        return out

    def partial(self, cycles):
        ti, tc = _d(), _d()
        hist = np.zeros(cycles)
        if ref_lib().ref_mgrit_partial(self.h, cycles, C.byref(ti), C.byref(tc), _p(hist)):
            raise RuntimeError(_ref_err())
        return ti.value, tc.value, hist

    def initial(self):
        out = np.zeros(self.n)
        ref_lib().ref_mgrit_initial(self.h, _p(out))
        return out

    def load_terms(self):
        out = np.zeros((self.nt, self.n))
        has = ref_lib().ref_load_terms(self.h, _p(out))
        return out if has else None

    # ---- one phase at a time (mgrit.hpp:76-91, 185, 197-214)
    def initialize(self):
        g = _d()
        if ref_lib().ref_mgrit_initialize(self.h, C.byref(g)):
            raise RuntimeError(_ref_err())
        return g.value

    def mgrit_cycle(self, level=0):
        if ref_lib().ref_mgrit_cycle(self.h, level):
            raise RuntimeError(_ref_err())

    def residual_norm(self, level=0):
        v = _d()
        if ref_lib().ref_mgrit_residual_norm(self.h, level, C.byref(v)):
            raise RuntimeError(_ref_err())
        return v.value

    def points(self, level, which, k0, count):
        out = np.zeros((count, self.n))
        ref_lib().ref_mgrit_points(self.h, level, which, k0, count, _p(out))
        return out

    def residual_iters(self, level=0, workers=None):
        """Per-solve p-MG cycle counts of the residual wave at the current state."""
        steps = self.levels()[0][level]
        out = np.zeros(steps + 1, np.int32)
        if ref_lib().ref_mgrit_residual_iters(self.h, level, workers or (os.cpu_count() or 1), _p(out)):
            raise RuntimeError(_ref_err())
        return out

    def sequential(self):
        out = np.zeros((self.nt + 1, self.n))
        s, it = _ll(), _ll()
        if ref_lib().ref_sequential_integrate(self.h, _p(out), C.byref(s), C.byref(it)):
            raise RuntimeError(_ref_err())
        return out, s.value, it.value


# ---------------------------------------------------------------------------
# C restatement
# ---------------------------------------------------------------------------
class _OcCsr(C.Structure):
    _fields_ = [("n_rows", _i), ("n_cols", _i), ("row_offsets", _vp), ("col_indices", _vp),
                ("values", _vp)]


_oc = None


def oc_lib():
    global _oc
    if _oc is None:
        if not os.path.exists(OC_SO):
            raise RuntimeError(f"{OC_SO} missing: build it with `make -C oracle`")
        L = C.CDLL(OC_SO)
        L.oc_last_error.restype = C.c_char_p
        L.oc_spmv.argtypes = [_vp, _vp, _vp]
        L.oc_spmv_transpose.argtypes = [_vp, _vp, _vp]
        L.oc_gs_sweep.argtypes = [_vp, _vp, _vp, _i]
        L.oc_norm2.restype = _d
        L.oc_norm2.argtypes = [_vp, _i]
        L.oc_disc_create.restype = _vp
        L.oc_disc_create.argtypes = [_vp, _vp, _vp, _vp, _vp, _i, _vp, _vp, _vp]
        L.oc_disc_free.argtypes = [_vp]
        L.oc_hier_create.restype = _vp
        L.oc_hier_create.argtypes = [_vp, _d, _i, _i, _i, _i, _d, _i]
        L.oc_hier_free.argtypes = [_vp]
        L.oc_hier_csr.argtypes = [_vp, _i, _vp, _vp, _vp, _vp, _vp, _vp]
        L.oc_hier_n_levels.argtypes = [_vp]
        for f in ("oc_ilut_apply", "oc_restrict", "oc_prolong", "oc_hmg_wcycle", "oc_coarse_solve",
                  "oc_vcycle"):
            getattr(L, f).argtypes = [_vp, _vp, _vp]
        L.oc_solve.argtypes = [_vp, _vp, _vp, _d, _i, _i, _i, _vp, _vp, _vp, _vp, _i]
        L.oc_stepper_create.restype = _vp
        L.oc_stepper_create.argtypes = [_vp, _d, _d, _d, _d, _i, _i]
        L.oc_stepper_create_kind.restype = _vp
        L.oc_stepper_create_kind.argtypes = [_vp, _d, _d, _d, _i, _d, _i, _i]
        L.oc_stepper_free.argtypes = [_vp]
        L.oc_stepper_step.argtypes = [_vp, _vp, _vp, _vp, _vp, _vp]
        L.oc_sequential_integrate.argtypes = [_vp, _d, _d, _i, _d, _vp, _vp, _i, _d, _i, _vp, _vp,
                                              _vp]
        L.oc_mgrit_create.restype = _vp
        L.oc_mgrit_create.argtypes = [_vp, _d, _d, _i, _d, _vp, _vp, _i, _i, _i, _i, _d, _i, _i,
                                      _d, _i]
        L.oc_mgrit_create_kind.restype = _vp
        L.oc_mgrit_create_kind.argtypes = [_vp, _d, _d, _i, _d, _vp, _vp, _i, _i, _i, _i, _d, _i,
                                           _i, _i, _d, _i]
        L.oc_mgrit_free.argtypes = [_vp]
        L.oc_mgrit_levels.argtypes = [_vp, _vp, _vp]
        L.oc_mgrit_solve.argtypes = [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i]
        L.oc_mgrit_trajectory.argtypes = [_vp, _vp]
        _oc = L
    return _oc


def _oc_err():
    return oc_lib().oc_last_error().decode()


def _oc_struct(a: CSR, keep: list) -> _OcCsr:
    ro = np.ascontiguousarray(a.row_offsets, np.int32)
    ci = np.ascontiguousarray(a.col_indices, np.int32)
    v = np.ascontiguousarray(a.values, np.float64)
    keep += [ro, ci, v]
    return _OcCsr(a.n_rows, a.n_cols, _p(ro), _p(ci), _p(v))


def oc_spmv(a: CSR, x):
    keep = []
    s = _oc_struct(a, keep)
    x = np.ascontiguousarray(x, np.float64)
    y = np.zeros(a.n_rows)
    oc_lib().oc_spmv(C.byref(s), _p(x), _p(y))
    return y


def oc_spmv_transpose(a: CSR, x):
    keep = []
    s = _oc_struct(a, keep)
    x = np.ascontiguousarray(x, np.float64)
    y = np.zeros(a.n_cols)
    oc_lib().oc_spmv_transpose(C.byref(s), _p(x), _p(y))
    return y


def oc_gs_sweep(a: CSR, b, x, backward=False):
    keep = []
    s = _oc_struct(a, keep)
    x = np.array(x, np.float64, copy=True)
    if oc_lib().oc_gs_sweep(C.byref(s), _p(np.ascontiguousarray(b, np.float64)), _p(x),
                            int(backward)):
        raise RuntimeError(_oc_err())
    return x


class OcDisc:
    """Borrowed SpatialDiscretization arrays (pmultigrid.hpp:71-159) for the restatement."""

    def __init__(self, ops: dict):
        self.ops = ops
        self._keep = []
        k = self._keep
        self._mass = _oc_struct(ops["mass_p"], k)
        self._stiff = _oc_struct(ops["stiff_p"], k)
        self._tr = _oc_struct(ops["transfer"], k)
        self._ilp = np.ascontiguousarray(ops["inv_lumped_p"], np.float64)
        self._il1 = np.ascontiguousarray(ops["inv_lumped_1"], np.float64)
        nh = len(ops["h_mass"])
        self._hm = (_OcCsr * nh)(*[_oc_struct(a, k) for a in ops["h_mass"]])
        self._hs = (_OcCsr * nh)(*[_oc_struct(a, k) for a in ops["h_stiff"]])
        ne = max(nh - 1, 1)
        emb = [_oc_struct(a, k) for a in ops["h_embed"]] or [_OcCsr()]
        self._he = (_OcCsr * ne)(*emb)
        self.h = oc_lib().oc_disc_create(C.byref(self._mass), C.byref(self._stiff),
                                         C.byref(self._tr), _p(self._ilp), _p(self._il1), nh,
                                         self._hm, self._hs, self._he)
        self.n = ops["mass_p"].n_rows
        self.n1 = ops["transfer"].n_cols
        self.n_h = nh

    def __del__(self):
        if getattr(self, "h", None):
            oc_lib().oc_disc_free(self.h)


class OcHier:
    """Restated PMultigridHierarchy (pmultigrid.hpp:215-324)."""

    def __init__(self, disc: OcDisc, c, nu_pre=1, nu_post=1, gs_pre=2, gs_post=2, tau=1e-13,
                 fill=0):
        self.disc = disc
        self.n = disc.n
        self.h = oc_lib().oc_hier_create(disc.h, c, nu_pre, nu_post, gs_pre, gs_post, tau, fill)
        if not self.h:
            raise RuntimeError(_oc_err())

    def __del__(self):
        if getattr(self, "h", None):
            oc_lib().oc_hier_free(self.h)

    def csr(self, which):
        return _fetch_csr(oc_lib().oc_hier_csr, self.h, which)

    def _call(self, fn, a, n_out, inout=None):
        a = np.ascontiguousarray(a, np.float64)
        out = np.zeros(n_out) if inout is None else np.array(inout, np.float64, copy=True)
        rc = getattr(oc_lib(), fn)(self.h, _p(a), _p(out))
        if rc:
            raise RuntimeError(_oc_err())
        return out

    def ilut_apply(self, r):
        return self._call("oc_ilut_apply", r, self.n)

    def restrict(self, r):
        return self._call("oc_restrict", r, self.disc.n1)

    def prolong(self, e1):
        return self._call("oc_prolong", e1, self.n)

    def hmg_wcycle(self, b1, x1=None):
        return self._call("oc_hmg_wcycle", b1, len(b1), np.zeros(len(b1)) if x1 is None else x1)

    def coarse_solve(self, b):
        return self._call("oc_coarse_solve", b, len(b))

    def vcycle(self, b, x):
        return self._call("oc_vcycle", b, self.n, x)

    def solve(self, b, x0=None, rel_tol=1e-12, max_iter=400, fixed_cycles=0):
        b = np.ascontiguousarray(b, np.float64)
        x = np.zeros(self.n) if x0 is None else np.array(x0, np.float64, copy=True)
        it, conv, fr = _i(), _i(), _d()
        hist = np.zeros(max(max_iter, fixed_cycles, 1))
        if oc_lib().oc_solve(self.h, _p(b), _p(x), rel_tol, max_iter, fixed_cycles,
                             int(x0 is None), C.byref(it), C.byref(conv), C.byref(fr), _p(hist),
                             hist.size):
            raise RuntimeError(_oc_err())
        return {"x": x, "iterations": it.value, "converged": bool(conv.value),
                "final_relative_residual": fr.value, "residual_history": hist[: it.value].copy()}


class OcStepper:
    """Restated ThetaStepper (theta.hpp:92-146); kind 0 p-multigrid, 1 Jacobi CG."""

    def __init__(self, disc: OcDisc, kappa, dt, theta, rel_tol=1e-12, max_iter=400,
                 fixed_cycles=0, kind=0):
        self.disc = disc
        self.h = oc_lib().oc_stepper_create_kind(disc.h, kappa, dt, theta, kind, rel_tol, max_iter,
                                                 fixed_cycles)
        if not self.h:
            raise RuntimeError(_oc_err())

    def __del__(self):
        if getattr(self, "h", None):
            oc_lib().oc_stepper_free(self.h)

    def step(self, u_prev, load=None, guess=None):
        u_prev = np.ascontiguousarray(u_prev, np.float64)
        load = None if load is None else np.ascontiguousarray(load, np.float64)
        guess = None if guess is None else np.ascontiguousarray(guess, np.float64)
        out = np.zeros(self.disc.n)
        it = _i()
        rc = oc_lib().oc_stepper_step(self.h, _p(u_prev), _p(load), _p(guess), _p(out),
                                      C.byref(it))
        if rc:
            raise RuntimeError(_oc_err())
        return out, it.value


def oc_sequential_integrate(disc: OcDisc, nt, *, kappa=1.0, t_final=0.1, theta=1.0, u0=None,
                            loads=None, load_steady=False, rel_tol=1e-12, max_iter=400):
    u0 = None if u0 is None else np.ascontiguousarray(u0, np.float64)
    loads = None if loads is None else np.ascontiguousarray(loads, np.float64)
    traj = np.zeros((nt + 1, disc.n))
    s, it = _ll(), _ll()
    if oc_lib().oc_sequential_integrate(disc.h, kappa, t_final, nt, theta, _p(u0), _p(loads),
                                        int(load_steady), rel_tol, max_iter, _p(traj),
                                        C.byref(s), C.byref(it)):
        raise RuntimeError(_oc_err())
    return traj, s.value, it.value


class OcMgrit:
    """Restated MgritSolver (mgrit.hpp:50-331) with given u0 / load terms."""

    def __init__(self, disc: OcDisc, nt, *, kappa=1.0, t_final=0.1, theta=1.0, u0=None,
                 loads=None, load_steady=False, cycle=CYCLE_V, relax=RELAX_FCF, m=2,
                 halt_tol=1e-10, max_iter=50, coarse_floor=8, rel_tol=1e-12, sp_max_iter=400,
                 spatial_kind=0):
        self.disc = disc
        self.nt = nt
        self.max_iter = max_iter
        self._u0 = None if u0 is None else np.ascontiguousarray(u0, np.float64)
        self._loads = None if loads is None else np.ascontiguousarray(loads, np.float64)
        self.h = oc_lib().oc_mgrit_create_kind(disc.h, kappa, t_final, nt, theta, _p(self._u0),
                                               _p(self._loads), int(load_steady), cycle, relax, m,
                                               halt_tol, max_iter, coarse_floor, spatial_kind,
                                               rel_tol, sp_max_iter)
        if not self.h:
            raise RuntimeError(_oc_err())

    def __del__(self):
        if getattr(self, "h", None):
            oc_lib().oc_mgrit_free(self.h)

    def levels(self):
        steps = np.zeros(32, np.int32)
        dts = np.zeros(32)
        L = oc_lib().oc_mgrit_levels(self.h, _p(steps), _p(dts))
        return [int(s) for s in steps[:L]], [float(d) for d in dts[:L]]

    def solve(self):
        it, conv, gn, fr, solves, mi = _i(), _i(), _d(), _d(), _ll(), _d()
        hist = np.zeros(self.max_iter)
        if oc_lib().oc_mgrit_solve(self.h, C.byref(it), C.byref(conv), C.byref(gn), C.byref(fr),
                                   C.byref(solves), C.byref(mi), _p(hist), hist.size):
            raise RuntimeError(_oc_err())
        return {"iterations": it.value, "converged": bool(conv.value), "g_norm": gn.value,
                "final_relative_residual": fr.value, "total_spatial_solves": solves.value,
                "mean_spatial_iterations": mi.value, "residual_history": hist[: it.value].copy()}

    def trajectory(self):
        out = np.zeros((self.nt + 1, self.disc.n))
        oc_lib().oc_mgrit_trajectory(self.h, _p(out))
        return out
