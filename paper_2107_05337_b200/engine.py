"""Python mirror of the reference operator API over the engine's C ABI.

Class and method names follow ``/root/reference/proj/include/miga``
(``SpatialDiscretization``, ``PMultigridHierarchy``, ``ThetaStepper``,
``MgritSolver``, ``sequential_integrate``) so the parity tests read like the
reference's own Catch2 suites.  Everything below calls
``_lib/libphi_engine.so`` (include/phi_engine.h); there is no Python or CPU
compute path: if the library or the GPU is missing, calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_lib_trace" if os.environ.get("PHI_TRACE") == "1"
                        else ("_lib_" + os.environ["PHI_VARIANT"] if os.environ.get("PHI_VARIANT") else "_lib"),
                        "libphi_engine.so")

PHI_OK, PHI_ERR_INVALID, PHI_ERR_NOT_CONVERGED, PHI_ERR_CUDA, PHI_ERR_RUNTIME = range(5)
SOURCE_CONSTANT, SOURCE_SIN_EXP, SOURCE_SIN = 0, 1, 2
INIT_ZERO, INIT_SIN, INIT_COEFFS = 0, 1, 2
CYCLE_V, CYCLE_F, CYCLE_TWO_LEVEL = 0, 1, 2
RELAX_F, RELAX_FCF = 0, 1

# every symbol include/phi_engine.h declares (checked by tests/test_capi_cpu.py)
EXPORTED = [
    "phi_last_error", "phi_default_solver_config", "phi_default_mgrit_config", "phi_default_problem",
    "phi_device_count", "phi_set_device", "phi_synchronize", "phi_disc_build", "phi_disc_free",
    "phi_disc_info", "phi_disc_export", "phi_disc_vector", "phi_hier_create", "phi_hier_free",
    "phi_hier_export", "phi_hier_vcycle", "phi_hier_solve", "phi_hier_unit", "phi_hier_spmm", "phi_hier_time",
    "phi_stepper_create",
    "phi_stepper_free", "phi_stepper_step", "phi_sequential_integrate", "phi_mgrit_create",
    "phi_mgrit_free", "phi_mgrit_levels", "phi_mgrit_solve", "phi_mgrit_trajectory",
    "phi_mgrit_initial", "phi_mgrit_initialize", "phi_mgrit_cycle", "phi_mgrit_residual_norm",
    "phi_mgrit_launches", "phi_mgrit_set_init_coeffs", "phi_mgrit_profile", "phi_mgrit_wave_report",
    "phi_dev_tuning", "phi_dev_trace", "phi_setup_tables_1d", "phi_setup_dense_lu", "phi_setup_level_steps", "phi_mgrit_set_range", "phi_mgrit_initialize_state",
    "phi_mgrit_gnorm_terms", "phi_mgrit_residual_terms", "phi_mgrit_phase", "phi_mgrit_points",
    "phi_mgrit_stats", "phi_mgrit_residual_iters", "phi_mgrit_wave_levels",
    "phi_hier_vcycle_bytes", "phi_comm_nccl_unique_id", "phi_comm_create_nccl", "phi_comm_create_ops", "phi_comm_free", "phi_mgrit_set_comm",
]


class EngineError(RuntimeError):
    """Raised for PHI_ERR_CUDA / PHI_ERR_RUNTIME."""


class NotConvergedError(RuntimeError):
    """PHI_ERR_NOT_CONVERGED (the reference's runtime_error from theta.hpp:116-118)."""


class PmgOptions(C.Structure):
    _fields_ = [("ilut_tau", C.c_double), ("ilut_fill", C.c_int), ("nu_pre", C.c_int),
                ("nu_post", C.c_int), ("gs_pre", C.c_int), ("gs_post", C.c_int), ("exact", C.c_int)]


SOLVER_PMG, SOLVER_CG = 0, 1  # SpatialSolverKind (theta.hpp:64)


class SolverConfig(C.Structure):
    _fields_ = [("rel_tol", C.c_double), ("max_iter", C.c_int), ("fixed_cycles", C.c_int),
                ("pmg", PmgOptions), ("kind", C.c_int)]


class MgritConfig(C.Structure):
    _fields_ = [("cycle", C.c_int), ("relax", C.c_int), ("m", C.c_int), ("halt_tol", C.c_double),
                ("max_iter", C.c_int), ("coarse_floor", C.c_int)]


class Problem(C.Structure):
    _fields_ = [("kappa", C.c_double), ("t_final", C.c_double), ("theta", C.c_double),
                ("n_time_steps", C.c_int), ("source_kind", C.c_int), ("source_param", C.c_double),
                ("init_kind", C.c_int), ("init_coeffs", C.c_void_p), ("load_terms", C.c_void_p),
                ("load_terms_steady", C.c_int)]


class MgritResultC(C.Structure):
    _fields_ = [("iterations", C.c_int), ("converged", C.c_int), ("g_norm", C.c_double),
                ("final_relative_residual", C.c_double), ("total_spatial_solves", C.c_longlong),
                ("mean_spatial_iterations", C.c_double)]


_lib = None
_vp, _i, _d, _ll = C.c_void_p, C.c_int, C.c_double, C.c_longlong


def lib():
    """Load the engine library (fails loudly when it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise EngineError(f"{LIB_PATH} not built: run `python -m paper_2107_05337_b200.build`")
        L = C.CDLL(LIB_PATH)
        L.phi_last_error.restype = C.c_char_p
        L.phi_default_solver_config.argtypes = [_vp]
        L.phi_default_solver_config.restype = None
        L.phi_default_mgrit_config.argtypes = [_vp]
        L.phi_default_mgrit_config.restype = None
        L.phi_default_problem.argtypes = [_vp]
        L.phi_default_problem.restype = None
        L.phi_set_device.argtypes = [_i]
        L.phi_disc_build.argtypes = [_i, _i, _vp]
        L.phi_disc_free.argtypes = [_vp]
        L.phi_disc_free.restype = None
        L.phi_disc_info.argtypes = [_vp, _vp]
        L.phi_disc_export.argtypes = [_vp, _i, _vp, _vp, _vp, _vp, _vp, _vp]
        L.phi_disc_vector.argtypes = [_vp, _i, _vp]
        L.phi_hier_create.argtypes = [_vp, _d, _vp, _vp]
        L.phi_hier_free.argtypes = [_vp]
        L.phi_hier_free.restype = None
        L.phi_hier_export.argtypes = [_vp, _i, _vp, _vp, _vp, _vp, _vp, _vp]
        L.phi_hier_vcycle.argtypes = [_vp, _vp, _vp, _i, _ll, _i]
        L.phi_hier_solve.argtypes = [_vp, _vp, _vp, _i, _ll, _d, _i, _i, _i, _vp, _vp, _vp, _i]
        L.phi_hier_unit.argtypes = [_vp, _i, _i, _i, _vp, _i, _vp, _i]
        L.phi_hier_spmm.argtypes = [_vp, _vp, _vp, _i, _i]
        L.phi_hier_time.argtypes = [_vp, _i, _i, _i, _i, _vp]
        L.phi_hier_vcycle_bytes.argtypes = [_vp, _i, _vp]
        L.phi_stepper_create.argtypes = [_vp, _d, _d, _d, _vp, _vp]
        L.phi_stepper_free.argtypes = [_vp]
        L.phi_stepper_free.restype = None
        L.phi_stepper_step.argtypes = [_vp, _vp, _vp, _vp, _i, _ll, _i, _vp, _i]
        L.phi_sequential_integrate.argtypes = [_vp, _i, _vp, _vp, _i, _vp, _vp, _vp]
        L.phi_mgrit_create.argtypes = [_vp, _vp, _vp, _vp, _vp]
        L.phi_mgrit_free.argtypes = [_vp]
        L.phi_mgrit_free.restype = None
        L.phi_mgrit_levels.argtypes = [_vp, _vp, _vp]
        L.phi_mgrit_solve.argtypes = [_vp, _vp, _vp, _i]
        L.phi_mgrit_trajectory.argtypes = [_vp, _vp]
        L.phi_mgrit_initial.argtypes = [_vp, _vp]
        L.phi_mgrit_initialize.argtypes = [_vp, _vp]
        L.phi_mgrit_cycle.argtypes = [_vp, _i]
        L.phi_mgrit_residual_norm.argtypes = [_vp, _i, _vp]
        L.phi_mgrit_launches.argtypes = [_vp]
        L.phi_mgrit_launches.restype = _ll
        L.phi_dev_tuning.argtypes = [_i, _i, _i]
        L.phi_dev_trace.argtypes = [_vp, _i]
        L.phi_setup_tables_1d.argtypes = [_i, _i, _i, _vp, _vp, _vp, _vp, _vp]
        L.phi_setup_dense_lu.argtypes = [_i, _vp, _vp, _vp]
        L.phi_setup_level_steps.argtypes = [_i, _i, _i, _i, _vp, _i, _vp]
        L.phi_mgrit_set_range.argtypes = [_vp, _i, _i]
        L.phi_mgrit_initialize_state.argtypes = [_vp]
        L.phi_mgrit_gnorm_terms.argtypes = [_vp, _vp]
        L.phi_mgrit_residual_terms.argtypes = [_vp, _i, _vp]
        L.phi_mgrit_residual_iters.argtypes = [_vp, _i, _vp]
        L.phi_mgrit_wave_levels.argtypes = [_vp, _vp, _vp, _vp, _vp, _i]
        L.phi_comm_nccl_unique_id.argtypes = [_vp]
        L.phi_comm_create_nccl.argtypes = [_vp, _i, _i, _vp]
        L.phi_comm_create_ops.argtypes = [_vp, _i, _i, _vp]
        L.phi_comm_free.argtypes = [_vp]
        L.phi_comm_free.restype = None
        L.phi_mgrit_set_comm.argtypes = [_vp, _vp]
        L.phi_mgrit_phase.argtypes = [_vp, _i, _i]
        L.phi_mgrit_points.argtypes = [_vp, _i, _i, _i, _i, _vp, _i, _i]
        L.phi_mgrit_stats.argtypes = [_vp, _vp]
        L.phi_mgrit_set_init_coeffs.argtypes = [_vp, _vp]
        L.phi_mgrit_profile.argtypes = [_vp, _i]
        L.phi_mgrit_wave_report.argtypes = [_vp, _vp, _vp]
        _lib = L
    return _lib


def _check(rc: int) -> None:
    if rc == PHI_OK:
        return
    msg = lib().phi_last_error().decode()
    if rc == PHI_ERR_INVALID:
        raise ValueError(msg)
    if rc == PHI_ERR_NOT_CONVERGED:
        raise NotConvergedError(msg)
    raise EngineError(msg)


def _p(a):
    return None if a is None else a.ctypes.data_as(_vp)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def dev_tuning(tri_warps=16, gs_warps=16, sleep_ns=0) -> None:
    """Developer knob for the sync-free sweeps (see include/phi_engine.h)."""
    _check(lib().phi_dev_tuning(tri_warps, gs_warps, sleep_ns))


def setup_tables_1d(degree: int, n_elements: int, nq: int) -> dict:
    """Host quadrature / basis tables of one parametric direction (no device
    needed): DirTables of an open uniform knot vector (assembly.hpp:124-151)."""
    pts = n_elements * nq
    out = dict(nodes=np.empty(pts), weights=np.empty(pts), vals=np.empty((pts, degree + 1)),
               ders=np.empty((pts, degree + 1)), first=np.empty(n_elements, dtype=np.int32))
    if degree < 1 or n_elements < 1 or nq < 1:  # the library raises; nothing to size
        out = {k: np.empty(1, dtype=v.dtype) for k, v in out.items()}
    _check(lib().phi_setup_tables_1d(degree, n_elements, nq, _p(out["nodes"]), _p(out["weights"]), _p(out["vals"]),
                                     _p(out["ders"]), _p(out["first"])))
    return out


def setup_dense_lu(a) -> tuple[np.ndarray, np.ndarray]:
    """DenseLU factors (unit-lower and upper packed) and permutation (solvers.hpp:136-167)."""
    a = _f64(a)
    if a.ndim != 2 or a.shape[0] != a.shape[1]:
        raise ValueError("DenseLU: matrix not square")
    n = a.shape[0]
    lu = np.empty((n, n))
    piv = np.empty(n, dtype=np.int32)
    _check(lib().phi_setup_dense_lu(n, _p(a), _p(lu), _p(piv)))
    return lu, piv


def setup_level_steps(nt: int, m: int, cycle: int = 0, coarse_floor: int = 8) -> list[int]:
    """Step counts of the MGRIT time levels (MgritSolver::build_levels, mgrit.hpp:217-233)."""
    steps = np.zeros(64, dtype=np.int32)
    nl = C.c_int(0)
    _check(lib().phi_setup_level_steps(nt, m, cycle, coarse_floor, _p(steps), 64, C.byref(nl)))
    return [int(v) for v in steps[: nl.value]]


def default_solver_config(**kw) -> SolverConfig:
    """SpatialSolverConfig (theta.hpp:66-75); kind=SOLVER_CG selects the Jacobi CG."""
    c = SolverConfig()
    lib().phi_default_solver_config(C.byref(c))
    for k, v in kw.items():
        if k in ("ilut_tau", "ilut_fill", "nu_pre", "nu_post", "gs_pre", "gs_post", "exact"):
            setattr(c.pmg, k, int(v) if k == "exact" else v)
        else:
            setattr(c, k, v)
    return c


@dataclass
class CSR:
    """Mirror of miga::SparseMatrix (sparse.hpp:17-22)."""

    n_rows: int
    n_cols: int
    row_offsets: np.ndarray
    col_indices: np.ndarray
    values: np.ndarray

    @property
    def nnz(self) -> int:
        return int(self.col_indices.size)


def _fetch(fn, h, which) -> CSR:
    nr, nc, nnz = _i(), _i(), _i()
    _check(fn(h, which, C.byref(nr), C.byref(nc), C.byref(nnz), None, None, None))
    ro = np.zeros(nr.value + 1, np.int32)
    ci = np.zeros(nnz.value, np.int32)
    v = np.zeros(nnz.value)
    _check(fn(h, which, None, None, None, _p(ro), _p(ci), _p(v)))
    return CSR(nr.value, nc.value, ro, ci, v)


class SpatialDiscretization:
    """SpatialDiscretization::build(unit_square, degree, mesh_exponent) (pmultigrid.hpp:94-158),
    assembled on the device."""

    def __init__(self, handle):
        self.h = handle
        info = np.zeros(5, np.int32)
        _check(lib().phi_disc_info(self.h, _p(info)))
        self.n_free, self.n_free_1, self.n_h_levels, self.n_elements, self.degree = map(int, info)

    @classmethod
    def build(cls, degree: int, mesh_exponent: int) -> "SpatialDiscretization":
        h = _vp()
        _check(lib().phi_disc_build(degree, mesh_exponent, C.byref(h)))
        return cls(h)

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.phi_disc_free(self.h)
            self.h = None

    def csr(self, which: int) -> CSR:
        return _fetch(lib().phi_disc_export, self.h, which)

    def vec(self, which: int) -> np.ndarray:
        out = np.zeros(self.n_free if which == 0 else self.n_free_1)
        _check(lib().phi_disc_vector(self.h, which, _p(out)))
        return out

    def operators(self) -> dict:
        return {
            "mass_p": self.csr(0), "stiff_p": self.csr(1), "transfer": self.csr(2),
            "inv_lumped_p": self.vec(0), "inv_lumped_1": self.vec(1),
            "h_mass": [self.csr(100 + l) for l in range(self.n_h_levels)],
            "h_stiff": [self.csr(200 + l) for l in range(self.n_h_levels)],
            "h_embed": [self.csr(300 + l) for l in range(self.n_h_levels - 1)],
        }


class PMultigridHierarchy:
    """PMultigridHierarchy(disc, c, opt) (pmultigrid.hpp:215-324), device resident."""

    def __init__(self, disc: SpatialDiscretization, c: float, nu_pre=1, nu_post=1, gs_pre=2,
                 gs_post=2, ilut_tau=1e-13, ilut_fill=0, exact=False):
        """exact=True: the reference's summation order (bit-identical results);
        False: reassociated parallel sums (within the solver tolerance)."""
        self.disc = disc
        self.n = disc.n_free
        opt = PmgOptions(ilut_tau, ilut_fill, nu_pre, nu_post, gs_pre, gs_post, int(exact))
        self.h = _vp()
        _check(lib().phi_hier_create(disc.h, c, C.byref(opt), C.byref(self.h)))

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.phi_hier_free(self.h)
            self.h = None

    def csr(self, which: int) -> CSR:
        return _fetch(lib().phi_hier_export, self.h, which)

    def vcycle(self, b, x) -> np.ndarray:
        b = _f64(b)
        x = np.array(x, dtype=np.float64, copy=True, order="C")
        nrhs = 1 if b.ndim == 1 else b.shape[0]
        _check(lib().phi_hier_vcycle(self.h, _p(b), _p(x), nrhs, self.n, 0))
        return x

    def solve(self, b, x0=None, rel_tol=1e-12, max_iter=400, fixed_cycles=0):
        b = _f64(b)
        nrhs = 1 if b.ndim == 1 else b.shape[0]
        x = np.zeros_like(b) if x0 is None else np.array(x0, dtype=np.float64, copy=True, order="C")
        it = np.zeros(nrhs, np.int32)
        cv = np.zeros(nrhs, np.int32)
        fr = np.zeros(nrhs)
        _check(lib().phi_hier_solve(self.h, _p(b), _p(x), nrhs, self.n, rel_tol, max_iter,
                                    fixed_cycles, int(x0 is None), _p(it), _p(cv), _p(fr), 0))
        if b.ndim == 1:
            return {"x": x, "iterations": int(it[0]), "converged": bool(cv[0]),
                    "final_relative_residual": float(fr[0])}
        return {"x": x, "iterations": it, "converged": cv.astype(bool),
                "final_relative_residual": fr}

    def _unit(self, op, vin, n_out, out=None, arg=0, arg2=0):
        vin = _f64(vin)
        o = np.zeros(n_out) if out is None else np.array(out, dtype=np.float64, copy=True)
        _check(lib().phi_hier_unit(self.h, op, arg, arg2, _p(vin), vin.size, _p(o), o.size))
        return o

    def spmm(self, X):
        """Y = A_p X for X of shape (n, nrhs), nrhs in {1, 16, 32, 64} (batched
        spmv, sparse.hpp:114-124; right-hand sides contiguous)."""
        X = np.ascontiguousarray(X, np.float64)
        nrhs = 1 if X.ndim == 1 else X.shape[1]
        Y = np.empty_like(X)
        _check(lib().phi_hier_spmm(self.h, _p(X), _p(Y), nrhs, 0))
        return Y

    def time_kernel(self, which: int, nrhs: int, reps: int = 5, flush_l2: int = 1) -> float:
        """Average device ms of one SpMM (which 0) or one V-cycle from x0 = 0
        (which 1) on nrhs seeded N(0,1) right-hand sides (BASELINE config 5).
        flush_l2 1: L2 flushed, events around each launch; 2 (SpMM): back-to-back
        launches over four copies of the operator (phi_hier_time)."""
        ms = C.c_double()
        _check(lib().phi_hier_time(self.h, which, nrhs, reps, int(flush_l2), C.byref(ms)))
        return ms.value

    def vcycle_bytes(self, nrhs: int) -> float:
        """Algorithmic bytes of one V-cycle on nrhs right-hand sides."""
        v = _d()
        _check(lib().phi_hier_vcycle_bytes(self.h, nrhs, C.byref(v)))
        return v.value

    def spmv(self, x):
        return self._unit(0, x, self.n)

    def ilut_apply(self, r):
        return self._unit(1, r, self.n)

    def restrict_to_linear(self, r):
        return self._unit(2, r, self.disc.n_free_1)

    def prolong_add(self, e1, x):
        return self._unit(3, e1, self.n, out=x)

    def prolong_from_linear(self, e1):
        return self._unit(3, e1, self.n, out=np.zeros(self.n))

    def hmg_wcycle(self, b1, x1=None):
        return self._unit(4, b1, len(b1), out=np.zeros(len(b1)) if x1 is None else x1)

    def gauss_seidel_sweep(self, level, b, x, backward=False):
        return self._unit(5, b, len(b), out=x, arg=level, arg2=int(backward))


class ThetaStepper:
    """ThetaStepper(disc, kappa, dt, theta, cfg) (theta.hpp:92-146)."""

    def __init__(self, disc: SpatialDiscretization, kappa: float, dt: float, theta: float,
                 cfg: SolverConfig | None = None):
        self.disc = disc
        self.n = disc.n_free
        cfg = cfg or default_solver_config()
        self.h = _vp()
        _check(lib().phi_stepper_create(disc.h, kappa, dt, theta, C.byref(cfg), C.byref(self.h)))

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.phi_stepper_free(self.h)
            self.h = None

    def step(self, u_prev, load=None, guess=None):
        """Batched: u_prev (nrhs, n) or (n,); returns Phi(u_prev) + load."""
        u = _f64(u_prev)
        nrhs = 1 if u.ndim == 1 else u.shape[0]
        ld = None if load is None else _f64(np.broadcast_to(load, u.shape))
        x = np.zeros_like(u) if guess is None else np.array(np.broadcast_to(guess, u.shape),
                                                              dtype=np.float64, order="C")
        it = np.zeros(nrhs, np.int32)
        _check(lib().phi_stepper_step(self.h, _p(u), _p(ld), _p(x), nrhs, self.n,
                                      int(guess is None), _p(it), 0))
        return x

    def sequential_integrate(self, nt, u0=None, loads=None, load_steady=False):
        traj = np.zeros((nt + 1, self.n))
        u0 = None if u0 is None else _f64(u0)
        loads = None if loads is None else _f64(loads)
        s, it = _ll(), _ll()
        _check(lib().phi_sequential_integrate(self.h, nt, _p(u0), _p(loads), int(load_steady),
                                              _p(traj), C.byref(s), C.byref(it)))
        return traj, s.value, it.value


@dataclass
class MgritResult:
    """MgritResult (mgrit.hpp:33-42), free-dof trajectory."""

    iterations: int
    converged: bool
    g_norm: float
    final_relative_residual: float
    total_spatial_solves: int
    mean_spatial_iterations: float
    residual_history: np.ndarray = field(repr=False)


_SHIFT = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_longlong)
_GATHER = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_longlong)


class CommOps(C.Structure):
    _fields_ = [("ctx", C.c_void_p), ("shift", _SHIFT), ("allgather", _GATHER)]


class Comm:
    """A rank of the time partition (phi_comm, include/phi_engine.h): attach
    with MgritSolver.set_comm and solve() runs the sharded schedule in the
    engine.  Comm.nccl(id, nranks, rank): NCCL over NVLink; Comm.ops(shift,
    allgather, nranks, rank): host callbacks on numpy arrays."""

    def __init__(self, handle, keep=None):
        self.h = handle
        self._keep = keep

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_ubyte * 128)()
        _check(lib().phi_comm_nccl_unique_id(buf))
        return bytes(buf)

    @classmethod
    def nccl(cls, uid: bytes, nranks: int, rank: int) -> "Comm":
        buf = (C.c_ubyte * 128).from_buffer_copy(uid)
        h = _vp()
        _check(lib().phi_comm_create_nccl(buf, nranks, rank, C.byref(h)))
        return cls(h)

    @classmethod
    def ops(cls, shift, allgather, nranks: int, rank: int) -> "Comm":
        """shift(send | None, count) -> recv | None; allgather(send) -> all
        (numpy float64 arrays)."""
        def _shift(_ctx, send, recv, count):
            try:
                s = np.ctypeslib.as_array(send, (count,)).copy() if send else None
                r = shift(s, count)
                if recv:
                    np.ctypeslib.as_array(recv, (count,))[:] = r
                return 0
            except Exception:  # reported to the engine as a transport failure
                return 1

        def _gather(_ctx, send, recv, count):
            try:
                a = allgather(np.ctypeslib.as_array(send, (count,)).copy())
                np.ctypeslib.as_array(recv, (count * nranks,))[:] = a
                return 0
            except Exception:
                return 1

        ops = CommOps(None, _SHIFT(_shift), _GATHER(_gather))
        h = _vp()
        _check(lib().phi_comm_create_ops(C.byref(ops), nranks, rank, C.byref(h)))
        return cls(h, keep=ops)

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.phi_comm_free(self.h)
            self.h = None


class MgritSolver:
    """MgritSolver(disc, ps, cfg, scfg) (mgrit.hpp:50-320); space-time state on device."""

    def __init__(self, disc: SpatialDiscretization, nt: int, *, kappa=1.0, t_final=0.1, theta=1.0,
                 source_kind=SOURCE_CONSTANT, source_param=1.0, init_kind=INIT_ZERO,
                 init_coeffs=None, load_terms=None, load_terms_steady=False, cycle=CYCLE_V,
                 relax=RELAX_FCF, m=2, halt_tol=1e-10, max_iter=50, coarse_floor=8,
                 solver: SolverConfig | None = None, exact: bool | None = None):
        self.disc = disc
        self.nt = nt
        self.max_iter = max_iter
        self.m, self.cycle, self.relax, self.halt_tol = m, cycle, relax, halt_tol
        self._coeffs = None if init_coeffs is None else _f64(init_coeffs)
        self._loads = None if load_terms is None else _f64(load_terms)
        ps = Problem(kappa, t_final, theta, nt, source_kind, source_param, init_kind,
                     None if self._coeffs is None else self._coeffs.ctypes.data,
                     None if self._loads is None else self._loads.ctypes.data, int(load_terms_steady))
        cfg = MgritConfig(cycle, relax, m, halt_tol, max_iter, coarse_floor)
        scfg = solver or default_solver_config()
        if exact is not None:
            scfg.pmg.exact = int(exact)
        self.h = _vp()
        _check(lib().phi_mgrit_create(disc.h, C.byref(ps), C.byref(cfg), C.byref(scfg),
                                      C.byref(self.h)))

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.phi_mgrit_free(self.h)
            self.h = None

    def levels(self):
        steps = np.zeros(32, np.int32)
        dts = np.zeros(32)
        L = lib().phi_mgrit_levels(self.h, _p(steps), _p(dts))
        return [int(s) for s in steps[:L]], [float(d) for d in dts[:L]]

    def solve(self) -> MgritResult:
        r = MgritResultC()
        hist = np.zeros(self.max_iter)
        _check(lib().phi_mgrit_solve(self.h, C.byref(r), _p(hist), hist.size))
        return MgritResult(r.iterations, bool(r.converged), r.g_norm, r.final_relative_residual,
                           r.total_spatial_solves, r.mean_spatial_iterations,
                           hist[: r.iterations].copy())

    def trajectory(self) -> np.ndarray:
        out = np.zeros((self.nt + 1, self.disc.n_free))
        _check(lib().phi_mgrit_trajectory(self.h, _p(out)))
        return out

    def initial(self) -> np.ndarray:
        out = np.zeros(self.disc.n_free)
        _check(lib().phi_mgrit_initial(self.h, _p(out)))
        return out

    def initialize(self) -> float:
        g = _d()
        _check(lib().phi_mgrit_initialize(self.h, C.byref(g)))
        return g.value

    def mgrit_cycle(self, level=0) -> None:
        _check(lib().phi_mgrit_cycle(self.h, level))

    def residual_norm(self, level=0) -> float:
        v = _d()
        _check(lib().phi_mgrit_residual_norm(self.h, level, C.byref(v)))
        return v.value

    def launches(self) -> int:
        return int(lib().phi_mgrit_launches(self.h))

    # ---- phase-level access for the time-sharded driver (timeshard.py) ----
    def set_range(self, j_lo: int, j_hi: int) -> None:
        _check(lib().phi_mgrit_set_range(self.h, j_lo, j_hi))

    def initialize_state(self) -> None:
        _check(lib().phi_mgrit_initialize_state(self.h))

    def gnorm_terms(self) -> np.ndarray:
        out = np.zeros(self.levels()[0][0] + 1)
        _check(lib().phi_mgrit_gnorm_terms(self.h, _p(out)))
        return out

    def residual_terms(self, level: int = 0) -> np.ndarray:
        out = np.zeros(self.levels()[0][level] + 1)
        _check(lib().phi_mgrit_residual_terms(self.h, level, _p(out)))
        return out

    def set_comm(self, comm: "Comm | None") -> None:
        """Shard level 0 over the communicator's ranks (None: one process)."""
        self._comm = comm
        _check(lib().phi_mgrit_set_comm(self.h, comm.h if comm is not None else None))

    def residual_iters(self, level: int = 0) -> np.ndarray:
        """Per-solve p-MG cycle counts of the residual wave at the current state."""
        out = np.zeros(self.levels()[0][level] + 1, np.int32)
        _check(lib().phi_mgrit_residual_iters(self.h, level, _p(out)))
        return out

    def phase(self, level: int, op: int) -> None:
        _check(lib().phi_mgrit_phase(self.h, level, op))

    def points(self, level: int, which: int, k0: int, count: int, ptr: int, device: bool, set_: bool) -> None:
        _check(lib().phi_mgrit_points(self.h, level, which, k0, count, ptr, int(device), int(set_)))

    def stats(self) -> tuple[int, int, int, int]:
        out = np.zeros(4, np.int64)
        _check(lib().phi_mgrit_stats(self.h, _p(out)))
        return tuple(int(v) for v in out)

    def set_init_coeffs(self, coeffs) -> None:
        self._coeffs = _f64(coeffs)
        _check(lib().phi_mgrit_set_init_coeffs(self.h, _p(self._coeffs)))

    def set_profile(self, enable: bool) -> None:
        _check(lib().phi_mgrit_profile(self.h, int(enable)))

    def wave_levels(self, cap: int = 8):
        """Per level of the last profiled solve(): (ms, Phi solves, p-MG cycles,
        dependent steps of one single-RHS V-cycle).  Call before wave_report()."""
        ms = np.zeros(cap)
        pts, cyc, steps = (np.zeros(cap, np.int64) for _ in range(3))
        _check(lib().phi_mgrit_wave_levels(self.h, _p(ms), _p(pts), _p(cyc), _p(steps), cap))
        L = len(self.levels()[0])
        return [dict(level=l, ms=float(ms[l]), solves=int(pts[l]), cycles=int(cyc[l]), chain_steps=int(steps[l]))
                for l in range(L)]

    def wave_report(self):
        """(waves, kernel ms, algorithmic bytes) of the last profiled solve()."""
        ms, by = _d(), _d()
        n = lib().phi_mgrit_wave_report(self.h, C.byref(ms), C.byref(by))
        if n < 0:
            _check(-n)
        return n, ms.value, by.value
