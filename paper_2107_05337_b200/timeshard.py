"""Time-sharded MGRIT over ranks (one process per GPU) -- SURVEY.md section 8(e).

Time shards naturally, space does not: every rank holds full replicas of the
operators and of the space-time arrays, and owns a contiguous block of the
coarse intervals of level 0 (`partition`).  Per MGRIT iteration
(mgrit.hpp:93-118, 278-288):

  F / FC relaxation   local to the owned intervals; the first owned interval
                      starts from the C-point u[J0 m] that rank r-1 owns, so a
                      halo exchange (one n-vector, rank r-1 -> r) precedes
                      every relaxation sweep;
  restriction         local (each coarse point j+1 is restricted from the
                      owned interval j); every rank then gathers the other
                      ranks' coarse right-hand sides (an allgather of the owned
                      points only, padded to the largest share);
  coarse cycle        replicated on every rank (the serial coarse march is the
                      Amdahl term either way, and replication needs no
                      scatter); under the F-schedule the second pass runs its
                      coarse cycle without the schedule, as cycle_impl(l,
                      false) does (mgrit.hpp:278-288);
  correction          injection of the coarse correction (replicated), then a
                      local F-relaxation;
  residual norm       per-point squared residuals of the owned points, summed
                      elementwise over the ranks, then in point order on the
                      host: the same floating-point sum as one process.

The collectives go through torch.distributed (NCCL between GPUs, gloo for the
CPU tests).  A rank's compute goes through an *executor* with the phase-level
interface of the engine's C ABI (phi_mgrit_phase & co.); `EngineExecutor`
wraps the CUDA engine.  With identical inputs the sharded solve performs the
same floating-point operations as the single-process solve, so its results
are identical for any rank count.

The product path for N > 1 is the same schedule in the C++ host
(csrc/timeshard.cpp, phi_mgrit_set_comm): `nccl_comm_from_torch` builds its
NCCL communicator (the unique id travels over torch.distributed) and
MgritSolver.solve() then runs sharded inside the engine.  TimeShardedMgrit
below is the Python statement of that schedule over any phase-level
executor; the CPU tests drive it with an executor over the oracle.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch
import torch.distributed as dist

# phase ops of phi_mgrit_phase; OP_CYCLE runs cycle_impl(l, cycle == F),
# OP_CYCLE_NOF cycle_impl(l, false)
OP_F, OP_FC, OP_RESTRICT, OP_INJECT, OP_CYCLE, OP_CYCLE_NOF = range(6)
U, G = 0, 1


def nccl_comm_from_torch(group=None):
    """phi_comm over NCCL for this torch.distributed rank (one GPU per rank):
    rank 0 creates the NCCL unique id and broadcasts it."""
    from .engine import Comm
    rank, size = dist.get_rank(group), dist.get_world_size(group)
    box = [Comm.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(box, src=0, group=group)
    return Comm.nccl(box[0], size, rank)


def partition(n_intervals: int, n_ranks: int, rank: int) -> tuple[int, int]:
    """Contiguous, near-equal split of the coarse intervals: [j0, j1)."""
    base, extra = divmod(n_intervals, n_ranks)
    j0 = rank * base + min(rank, extra)
    return j0, j0 + base + (1 if rank < extra else 0)


class TorchComm:
    """The three exchanges the sharded cycle needs, over torch.distributed."""

    def __init__(self, device: torch.device, group=None):
        self.group = group
        self.rank = dist.get_rank(group)
        self.size = dist.get_world_size(group)
        self.device = device

    def shift(self, send: torch.Tensor | None, recv: torch.Tensor | None) -> None:
        """Rank r sends `send` to r+1 and receives `recv` from r-1."""
        ops = []
        if send is not None and self.rank + 1 < self.size:
            ops.append(dist.P2POp(dist.isend, send, self.rank + 1, self.group))
        if recv is not None and self.rank > 0:
            ops.append(dist.P2POp(dist.irecv, recv, self.rank - 1, self.group))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()

    def allreduce_sum(self, t: torch.Tensor) -> None:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)

    def allgather(self, t: torch.Tensor) -> torch.Tensor:
        """Every rank's `t` (same size on all ranks), concatenated in rank order."""
        out = torch.empty(self.size * t.numel(), dtype=t.dtype, device=t.device)
        if hasattr(dist, "all_gather_into_tensor") and t.is_cuda:
            dist.all_gather_into_tensor(out, t.contiguous(), group=self.group)
        else:
            dist.all_gather(list(out.chunk(self.size)), t.contiguous(), group=self.group)
        return out


@dataclass
class ShardedResult:
    iterations: int = 0
    converged: bool = False
    g_norm: float = 0.0
    final_relative_residual: float = 0.0
    residual_history: list = field(default_factory=list)
    total_spatial_solves: int = 0
    mean_spatial_iterations: float = 0.0


class TimeShardedMgrit:
    """MgritSolver::solve (mgrit.hpp:93-118) with level 0 sharded over ranks.

    `ex` is the rank's executor; `comm` a TorchComm (or any object with the
    same three methods).  cycle: 0 V, 1 F, 2 two-level; relax: 0 F, 1 FCF.
    """

    def __init__(self, ex, comm, *, cycle: int, relax: int, halt_tol: float, max_iter: int):
        self.ex, self.comm = ex, comm
        self.cycle, self.relax = cycle, relax
        self.halt_tol, self.max_iter = halt_tol, max_iter
        self.n, self.m = ex.n, ex.m
        self.steps = ex.steps
        if len(self.steps) < 2:
            raise ValueError("time sharding needs at least two MGRIT levels")
        if self.steps[0] % self.m:
            raise ValueError("time sharding needs steps divisible by m on level 0")
        self.J = self.steps[0] // self.m
        if comm.size > self.J:
            raise ValueError(f"{comm.size} ranks for {self.J} coarse intervals")
        self.j0, self.j1 = partition(self.J, comm.size, comm.rank)
        ex.set_range(self.j0, self.j1)

    # ---- exchanges ---------------------------------------------------------
    def halo(self) -> None:
        """u[j0 m] (the C-point that ends interval j0 - 1) from rank r - 1."""
        c = self.comm
        send = self.ex.get_points(0, U, self.j1 * self.m, 1) if c.rank + 1 < c.size else None
        recv = torch.empty(self.n, dtype=torch.float64, device=c.device) if c.rank > 0 else None
        c.shift(send, recv)
        if recv is not None:
            self.ex.set_points(0, U, self.j0 * self.m, recv)

    def combine_coarse_rhs(self) -> None:
        """Coarse g at points j + 1 of every rank's intervals: an allgather of
        the owned points (padded to the largest share), placed in rank order."""
        n, J, R = self.n, self.J, self.comm.size
        shares = [partition(J, R, r) for r in range(R)]
        width = max(b - a for a, b in shares)
        mine = torch.zeros(width * n, dtype=torch.float64, device=self.comm.device)
        own = self.j1 - self.j0
        if own:
            mine[:own * n] = self.ex.get_points(1, G, self.j0 + 1, own)
        parts = self.comm.allgather(mine).view(R, width * n)
        full = torch.cat([parts[r, :(b - a) * n] for r, (a, b) in enumerate(shares)])
        self.ex.set_points(1, G, 1, full)
        # restriction zeroes the coarse iterate at every restricted point
        self.ex.set_points(1, U, 1, torch.zeros(J * n, dtype=torch.float64, device=self.comm.device))

    def ordered_norm(self, terms: np.ndarray) -> float:
        t = torch.as_tensor(terms, dtype=torch.float64).to(self.comm.device)
        self.comm.allreduce_sum(t)
        total = 0.0
        for v in t.cpu().numpy():  # point order (mgrit.hpp:211-212)
            total += float(v)
        return float(np.sqrt(total))

    # ---- cycle (mgrit.hpp:278-288 at level 0) -------------------------------
    def cycle0(self, f_schedule: bool) -> None:
        ex = self.ex
        self.halo()
        if self.relax == 1:
            ex.phase(0, OP_FC)
            self.halo()
        ex.phase(0, OP_F)
        ex.phase(0, OP_RESTRICT)
        self.combine_coarse_rhs()
        ex.phase(1, OP_CYCLE if f_schedule else OP_CYCLE_NOF)  # replicated coarse cycle
        ex.phase(0, OP_INJECT)
        self.halo()
        ex.phase(0, OP_F)
        if f_schedule and len(self.steps) > 2:
            self.cycle0(False)

    def solve(self) -> ShardedResult:
        ex = self.ex
        ex.initialize_state()
        res = ShardedResult()
        res.g_norm = self.ordered_norm(ex.gnorm_terms())
        denom = res.g_norm if res.g_norm > 0.0 else 1.0
        for it in range(1, self.max_iter + 1):
            self.cycle0(self.cycle == 1)
            self.halo()
            rel = self.ordered_norm(ex.residual_terms(0)) / denom
            res.residual_history.append(rel)
            res.iterations = it
            if rel <= self.halt_tol:
                res.converged = True
                break
        res.final_relative_residual = res.residual_history[-1]
        s0, i0, sc, ic = ex.stats()
        t = torch.tensor([s0, i0], dtype=torch.float64, device=self.comm.device)
        self.comm.allreduce_sum(t)  # level-0 work is split; coarse work is replicated
        solves, iters = int(t[0].item()) + sc, int(t[1].item()) + ic
        res.total_spatial_solves = solves
        res.mean_spatial_iterations = iters / solves if solves else 0.0
        return res

    def trajectory(self) -> np.ndarray:
        """Level-0 trajectory assembled on every rank ((steps + 1) x n)."""
        n, m = self.n, self.m
        full = torch.zeros((self.steps[0] + 1) * n, dtype=torch.float64, device=self.comm.device)
        k0 = 0 if self.j0 == 0 else self.j0 * m + 1
        k1 = self.j1 * m
        full[k0 * n:(k1 + 1) * n] = self.ex.get_points(0, U, k0, k1 - k0 + 1)
        self.comm.allreduce_sum(full)
        return full.cpu().numpy().reshape(self.steps[0] + 1, n)


class EngineExecutor:
    """Executor over the CUDA engine (paper_2107_05337_b200.MgritSolver)."""

    def __init__(self, solver, device: torch.device):
        self.s = solver
        self.device = device
        self.n = solver.disc.n_free
        self.steps = solver.levels()[0]
        self.m = solver.m

    def set_range(self, j0: int, j1: int) -> None:
        self.s.set_range(j0, j1)

    def initialize_state(self) -> None:
        self.s.initialize_state()

    def gnorm_terms(self) -> np.ndarray:
        return self.s.gnorm_terms()

    def residual_terms(self, level: int) -> np.ndarray:
        return self.s.residual_terms(level)

    def phase(self, level: int, op: int) -> None:
        self.s.phase(level, op)

    def get_points(self, level: int, which: int, k0: int, count: int) -> torch.Tensor:
        t = torch.empty(count * self.n, dtype=torch.float64, device=self.device)
        if count:
            self.s.points(level, which, k0, count, t.data_ptr(), True, False)
        return t

    def set_points(self, level: int, which: int, k0: int, t: torch.Tensor) -> None:
        t = t.contiguous()
        if t.numel():
            torch.cuda.current_stream(self.device).synchronize()
            self.s.points(level, which, k0, t.numel() // self.n, t.data_ptr(), True, True)

    def stats(self) -> tuple[int, int, int, int]:
        return self.s.stats()
