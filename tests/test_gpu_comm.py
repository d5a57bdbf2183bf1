"""Time sharding in the C++ host (csrc/timeshard.cpp, phi_mgrit_set_comm):
the engine runs the sharded schedule itself -- halo shifts, allgathered
coarse right-hand sides, point-ordered reductions -- and must reproduce the
single-process solve bit for bit (iterations, residual history, g-norm,
solve counts, trajectory) for any rank count.

  * NCCL transport, world size 1 (one GPU here);
  * host-callback transport (phi_comm_ops), world size 2: two engines on
    this GPU driven from two threads, exchanging through host memory (no
    device-side waits between the ranks);
  * NCCL transport, world size 2, when two GPUs are visible.
"""
import threading

import numpy as np
import pytest

from tests.conftest import gpu_available

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]

E = pytest.importorskip("paper_2107_05337_b200.engine")

CASES = [
    # two-level, transient source, spline u0 (the config-2 shape, small)
    dict(p=3, k=5, nt=64, kw=dict(cycle=E.CYCLE_TWO_LEVEL, m=8, source_kind=E.SOURCE_SIN_EXP,
                                  source_param=2 * np.pi ** 2, init_kind=E.INIT_COEFFS)),
    # F-cycle over four levels (64/32/16/8)
    dict(p=2, k=4, nt=64, kw=dict(cycle=E.CYCLE_F, m=2, source_kind=E.SOURCE_SIN_EXP,
                                  source_param=2 * np.pi ** 2, init_kind=E.INIT_COEFFS)),
    # V-cycle, steady source, three levels
    dict(p=2, k=4, nt=128, kw=dict(cycle=E.CYCLE_V, m=4, source_kind=E.SOURCE_SIN, source_param=1.0,
                                   init_kind=E.INIT_SIN)),
]


def _solver(case, exact):
    p, k, nt = case["p"], case["k"], case["nt"]
    kw = dict(case["kw"])
    if kw.get("init_kind") == E.INIT_COEFFS:
        kw["init_coeffs"] = np.random.default_rng(12345).uniform(-1, 1, (2 ** k + p - 2) ** 2)
    return E.MgritSolver(E.SpatialDiscretization.build(p, k), nt, exact=exact, **kw)


def _same(r, t, r0, t0):
    assert r.iterations == r0.iterations and r.converged == r0.converged
    assert r.g_norm == r0.g_norm
    assert np.array_equal(r.residual_history, r0.residual_history)
    assert r.total_spatial_solves == r0.total_spatial_solves
    assert r.mean_spatial_iterations == r0.mean_spatial_iterations
    assert np.array_equal(t, t0)


@pytest.mark.parametrize("case", range(len(CASES)))
@pytest.mark.parametrize("exact", [True, False])
def test_nccl_world1_equals_solve(case, exact):
    c = CASES[case]
    s0 = _solver(c, exact)
    r0, t0 = s0.solve(), s0.trajectory()
    s1 = _solver(c, exact)
    comm = E.Comm.nccl(E.Comm.unique_id(), 1, 0)
    s1.set_comm(comm)
    r1 = s1.solve()
    _same(r1, s1.trajectory(), r0, t0)


class _Mailbox:
    """In-process transport of two ranks (host memory, thread barriers)."""

    def __init__(self, size):
        self.size = size
        self.slots = [None] * size
        self.bar = threading.Barrier(size, timeout=600)

    def shift(self, rank, send, count):
        self.slots[rank] = send
        self.bar.wait()
        out = self.slots[rank - 1] if rank > 0 else None
        self.bar.wait()
        return out

    def allgather(self, rank, send):
        self.slots[rank] = send
        self.bar.wait()
        out = np.concatenate(self.slots)
        self.bar.wait()
        return out


@pytest.mark.parametrize("case", range(len(CASES)))
@pytest.mark.parametrize("exact", [True, False])
def test_ops_world2_equals_solve(case, exact):
    c = CASES[case]
    s0 = _solver(c, exact)
    r0, t0 = s0.solve(), s0.trajectory()
    box = _Mailbox(2)
    solvers = [_solver(c, exact) for _ in range(2)]
    comms = [E.Comm.ops(lambda s, n, r=r: box.shift(r, s, n), lambda s, r=r: box.allgather(r, s), 2, r)
             for r in range(2)]
    for s, cm in zip(solvers, comms):
        s.set_comm(cm)
    out = [None, None]

    def run(r):
        try:
            res = solvers[r].solve()
            out[r] = (res, solvers[r].trajectory())
        except Exception as e:  # surfaced below
            out[r] = e
            box.bar.abort()

    th = [threading.Thread(target=run, args=(r,)) for r in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=900)
    for r in range(2):
        assert not isinstance(out[r], Exception), out[r]
        _same(out[r][0], out[r][1], r0, t0)


def _two_gpus():
    try:
        import torch
        return torch.cuda.device_count() >= 2
    except Exception:
        return False


def _nccl_rank(rank, uid, q):
    import paper_2107_05337_b200.engine as EE
    EE.lib().phi_set_device(rank)
    s = _solver(CASES[0], False)
    s.set_comm(EE.Comm.nccl(uid, 2, rank))
    r = s.solve()
    q.put((rank, r.iterations, list(r.residual_history), s.trajectory()))


@pytest.mark.skipif(not _two_gpus(), reason="needs two GPUs")
def test_nccl_world2_equals_solve():
    import torch.multiprocessing as mp
    s0 = _solver(CASES[0], False)
    r0, t0 = s0.solve(), s0.trajectory()
    uid = E.Comm.unique_id()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_nccl_rank, args=(r, uid, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=600) for _ in ps]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    for _, it, hist, traj in res:
        assert it == r0.iterations
        assert np.array_equal(np.asarray(hist), r0.residual_history)
        assert np.array_equal(traj, t0)
