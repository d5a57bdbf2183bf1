"""The time-sharded driver over the CUDA engine (one rank here; the two-rank
schedule is pinned on CPU by test_timeshard_gloo.py): identical results to
the engine's own single-process solve(), and to the reference."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist

from oracle import oracle as O
from tests.conftest import gpu_available

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]

E = pytest.importorskip("paper_2107_05337_b200.engine")
TS = pytest.importorskip("paper_2107_05337_b200.timeshard")


@pytest.fixture(scope="module")
def group():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield
    dist.destroy_process_group()


@pytest.mark.parametrize("exact,cycle,m", [(True, 2, 8), (False, 2, 8), (True, 1, 2), (False, 1, 2)])
def test_sharded_driver_equals_solve(group, exact, cycle, m):
    """cycle 1 (F) with m = 2: 64/32/16/8, four levels -- the F-schedule's
    second pass runs its coarse cycle without the schedule (OP_CYCLE_NOF)."""
    p, k, nt = 3, 5, 64
    coeffs = np.random.default_rng(12345).uniform(-1, 1, (2 ** k + p - 2) ** 2)
    kw = dict(cycle=cycle, m=m, source_kind=E.SOURCE_SIN_EXP, source_param=2 * np.pi ** 2,
              init_kind=E.INIT_COEFFS, init_coeffs=coeffs, exact=exact)
    d = E.SpatialDiscretization.build(p, k)
    ref = E.MgritSolver(d, nt, **kw)
    r0 = ref.solve()
    t0 = ref.trajectory()
    sol = E.MgritSolver(d, nt, **kw)
    drv = TS.TimeShardedMgrit(TS.EngineExecutor(sol, torch.device("cuda", 0)), TS.TorchComm(torch.device("cuda", 0)),
                              cycle=sol.cycle, relax=sol.relax, halt_tol=sol.halt_tol, max_iter=sol.max_iter)
    r1 = drv.solve()
    assert r1.iterations == r0.iterations and r1.converged == r0.converged
    assert r1.g_norm == r0.g_norm
    assert np.array_equal(np.asarray(r1.residual_history), r0.residual_history)
    assert r1.total_spatial_solves == r0.total_spatial_solves
    assert r1.mean_spatial_iterations == r0.mean_spatial_iterations
    assert np.array_equal(drv.trajectory(), t0)
    if exact and O.ref_available():
        rr = O.RefMgrit(p, k, nt, **{a: b for a, b in kw.items() if a != "exact"})
        rres = rr.solve()
        assert r1.iterations == rres["iterations"]
        assert np.array_equal(drv.trajectory(), rr.trajectory())
