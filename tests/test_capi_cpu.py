"""CPU tests of the C ABI (include/phi_engine.h): the library loads, exports
every declared entry point, mirrors the reference's defaults and error
mapping, and fails loudly -- never falls back to the CPU -- without a device."""
from __future__ import annotations

import ctypes as C
import os
import re

import pytest

import paper_2107_05337_b200 as P
from paper_2107_05337_b200 import engine as E

from .conftest import gpu_available

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "phi_engine.h")


def _declared() -> list[str]:
    text = re.sub(r"/\*.*?\*/", "", open(HEADER).read(), flags=re.S)
    return sorted(set(re.findall(r"\b(phi_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(E.LIB_PATH):
        from paper_2107_05337_b200 import build

        build.build()
    return P.lib()


def test_every_declared_symbol_is_exported(lib):
    names = _declared()
    assert len(names) >= 30
    for n in names:
        assert hasattr(lib, n), n
    assert sorted(E.EXPORTED) == names


def test_defaults_mirror_the_reference(lib):
    cfg = E.SolverConfig()
    lib.phi_default_solver_config(C.byref(cfg))
    # SpatialSolverConfig (theta.hpp:66-75), PMultigridOptions (pmultigrid.hpp:161-168)
    assert (cfg.rel_tol, cfg.max_iter, cfg.fixed_cycles) == (1e-12, 400, 0)
    o = cfg.pmg
    assert (o.ilut_tau, o.ilut_fill, o.nu_pre, o.nu_post, o.gs_pre, o.gs_post) == (1e-13, 0, 1, 1, 2, 2)
    m = E.MgritConfig()
    lib.phi_default_mgrit_config(C.byref(m))
    # MgritConfig (mgrit.hpp:17-31)
    assert (m.cycle, m.relax, m.m, m.halt_tol, m.max_iter, m.coarse_floor) == (0, 1, 2, 1e-10, 50, 8)
    ps = E.Problem()
    lib.phi_default_problem(C.byref(ps))
    # ProblemSpec (theta.hpp:42-62)
    assert (ps.kappa, ps.t_final, ps.theta, ps.n_time_steps) == (1.0, 0.1, 1.0, 64)
    assert (ps.source_kind, ps.source_param, ps.init_kind) == (E.SOURCE_CONSTANT, 1.0, E.INIT_ZERO)


def test_invalid_arguments_map_to_value_error(lib):
    out = C.c_void_p()
    assert lib.phi_disc_build(0, 3, C.byref(out)) == E.PHI_ERR_INVALID
    assert "degree" in lib.phi_last_error().decode()
    with pytest.raises(ValueError):
        P.SpatialDiscretization.build(2, 0)


@pytest.mark.skipif(gpu_available(), reason="checks the no-device behaviour")
def test_no_device_fails_loudly(lib):
    out = C.c_void_p()
    assert lib.phi_disc_build(2, 3, C.byref(out)) == E.PHI_ERR_CUDA
    assert lib.phi_last_error().decode()
    with pytest.raises(E.EngineError):
        P.SpatialDiscretization.build(2, 3)
