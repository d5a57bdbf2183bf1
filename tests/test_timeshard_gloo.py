"""Time-sharded MGRIT driver (paper_2107_05337_b200/timeshard.py) on CPU:
world size 2 over gloo, the rank's compute done by a restated executor over
the oracle's Phi (oracle.OcStepper -- test infrastructure), checked bit for
bit against the compiled reference's own MgritSolver results (golden
fixtures): iterations, residual history, g-norm, solve counts, trajectory.

This pins the sharding schedule itself -- interval partition, halo
exchanges, coarse right-hand-side combination, replicated coarse cycle and
the ordered cross-rank reductions -- independently of the GPU."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O
from paper_2107_05337_b200 import timeshard as TS

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")


def _seqdot(w):  # index-ordered sum of squares, as the reference's dot
    return float(np.cumsum(w * w)[-1]) if w.size else 0.0


class OracleExecutor:
    """Phase-level MGRIT restated over OcStepper (mgrit.hpp:122-214); the same
    operations in the same order as oracle/phi_oracle.c's solver."""

    def __init__(self, disc, nt, m, *, t_final=0.1, kappa=1.0, theta=1.0, u0=None, loads=None, cycle=2,
                 coarse_floor=8):
        self.n, self.m, self.cycle = disc.n, m, cycle
        steps = [nt]
        while True:
            cur = steps[-1]
            if cur % m or cur < m:
                break
            nxt = cur // m
            if len(steps) > 1 and nxt + 1 <= coarse_floor:
                break
            steps.append(nxt)
            if cycle == 2:
                break
        self.steps = steps
        dt0 = t_final / nt
        self.st = [O.OcStepper(disc, kappa, dt0 * (nt // s), theta) for s in steps]
        self.u0, self.loads = u0, loads
        self.u = [np.zeros((s + 1, self.n)) for s in steps]
        self.g = [np.zeros((s + 1, self.n)) for s in steps]
        self.j0, self.j1 = 0, steps[0] // m
        self.cnt = [0, 0, 0, 0]

    def set_range(self, j0, j1):
        self.j0, self.j1 = j0, j1

    def _rng(self, l):
        return (self.j0, self.j1) if l == 0 else (0, self.steps[l] // self.m)

    def _load(self, l, k):
        return None if (l != 0 or self.loads is None) else self.loads[k - 1]

    def _step_value(self, l, k):
        x, it = self.st[l].step(self.u[l][k - 1], self._load(l, k), self.u[l][k])
        self.cnt[0 if l == 0 else 2] += 1
        self.cnt[1 if l == 0 else 3] += it
        return x

    def _step_into(self, l, k):
        self.u[l][k] = self._step_value(l, k) + self.g[l][k]

    def initialize_state(self):
        for a in self.u + self.g:
            a[:] = 0.0
        if self.u0 is not None:
            self.g[0][0] = self.u0
            self.u[0][0] = self.u0
        self.cnt = [0, 0, 0, 0]

    def gnorm_terms(self):
        h = np.zeros(self.steps[0] + 1)
        if self.j0 == 0:
            h[0] = _seqdot(self.g[0][0])
        if self.loads is not None:
            for k in range(self.j0 * self.m + 1, self.j1 * self.m + 1):
                x, it = self.st[0].step(np.zeros(self.n), self.loads[k - 1], None)
                self.cnt[0] += 1
                self.cnt[1] += it
                h[k] = _seqdot(x)
        return h

    def residual_terms(self, l):
        h = np.zeros(self.steps[l] + 1)
        lo, hi = self._rng(l)
        if lo == 0:
            h[0] = _seqdot(self.g[l][0] - self.u[l][0])
        for k in range(lo * self.m + 1, hi * self.m + 1):
            w = self._step_value(l, k) + self.g[l][k]
            h[k] = _seqdot(w - self.u[l][k])
        return h

    def _f_relax(self, l, with_c):  # F-points of every interval, then (with_c) every C-point
        lo, hi = self._rng(l)
        for j in range(lo, hi):
            for t in range(1, self.m):
                self._step_into(l, j * self.m + t)
        if with_c:
            for j in range(lo, hi):
                self._step_into(l, (j + 1) * self.m)

    def _restrict(self, l):
        c = l + 1
        self.g[c][0] = self.g[l][0] - self.u[l][0]
        lo, hi = self._rng(l)
        for j in range(lo, hi):
            k = (j + 1) * self.m
            w = self._step_value(l, k) + self.g[l][k]
            self.g[c][j + 1] = w - self.u[l][k]
            self.u[c][j + 1] = 0.0
        self.u[c][0] = self.g[c][0]

    def _inject(self, l):
        for j in range(self.steps[l] // self.m + 1):
            self.u[l][j * self.m] = self.u[l][j * self.m] + self.u[l + 1][j]

    def _cycle(self, l, f_schedule):
        if l + 1 == len(self.steps):
            self.u[l][0] = self.g[l][0]
            for k in range(1, self.steps[l] + 1):
                self._step_into(l, k)
            return
        self._f_relax(l, True)  # FCF (the configurations tested here)
        self._f_relax(l, False)
        self._restrict(l)
        self._cycle(l + 1, f_schedule)
        self._inject(l)
        self._f_relax(l, False)
        if f_schedule and l + 2 < len(self.steps):
            self._cycle(l, False)

    def phase(self, l, op):
        if op == TS.OP_F:
            self._f_relax(l, False)
        elif op == TS.OP_FC:
            self._f_relax(l, True)
        elif op == TS.OP_RESTRICT:
            self._restrict(l)
        elif op == TS.OP_INJECT:
            self._inject(l)
        elif op == TS.OP_CYCLE_NOF:
            self._cycle(l, False)
        else:
            self._cycle(l, self.cycle == 1)

    def get_points(self, l, which, k0, count):
        a = self.u[l] if which == TS.U else self.g[l]
        return torch.from_numpy(a[k0:k0 + count].reshape(-1).copy())

    def set_points(self, l, which, k0, t):
        a = self.u[l] if which == TS.U else self.g[l]
        v = t.cpu().numpy().reshape(-1, self.n)
        a[k0:k0 + v.shape[0]] = v

    def stats(self):
        return tuple(self.cnt)


def _ops(g):
    def csr(prefix):
        nr, nc = (int(v) for v in g[prefix + "_shape"])
        return O.CSR(nr, nc, g[prefix + "_ro"], g[prefix + "_ci"], g[prefix + "_v"])
    nh = int(g["n_h"][0])
    return {"mass_p": csr("mass_p"), "stiff_p": csr("stiff_p"), "transfer": csr("transfer"),
            "inv_lumped_p": g["inv_lumped_p"], "inv_lumped_1": g["inv_lumped_1"],
            "h_mass": [csr(f"h_mass{l}") for l in range(nh)], "h_stiff": [csr(f"h_stiff{l}") for l in range(nh)],
            "h_embed": [csr(f"h_embed{l}") for l in range(nh - 1)]}


def _worker(rank, world, port, name, m, out, cycle=2):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = np.load(os.path.join(GOLD, name))
        nt = g["trajectory"].shape[0] - 1
        ex = OracleExecutor(O.OcDisc(_ops(g)), nt, m, u0=g["u0"], loads=g["loads"] if "loads" in g.files else None,
                            cycle=cycle)
        assert ex.steps == [int(v) for v in g["levels_steps"]]
        drv = TS.TimeShardedMgrit(ex, TS.TorchComm(torch.device("cpu")), cycle=cycle, relax=1, halt_tol=1e-10,
                                  max_iter=50)
        r = drv.solve()
        traj = drv.trajectory()
        if rank == 0:
            out.put((r.iterations, r.converged, r.g_norm, r.residual_history, r.total_spatial_solves,
                     r.mean_spatial_iterations, traj, (drv.j0, drv.j1)))
        else:
            out.put((drv.j0, drv.j1))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("name,m,cycle", [("mgrit_src.npz", 8, 2), ("mgrit_c1.npz", 4, 2),
                                          ("mgrit_fcycle.npz", 2, 1)])
def test_time_sharded_matches_reference_world2(name, m, cycle):
    """mgrit_fcycle: the F-schedule over 4 levels -- the second pass's coarse
    cycle must run without the schedule (OP_CYCLE_NOF), as in the reference."""
    if not os.path.exists(O.OC_SO):
        import subprocess
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, name, m, q, cycle)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    full = next(x for x in res if len(x) > 2)
    it, conv, gnorm, hist, solves, mean, traj, rng0 = full
    g = np.load(os.path.join(GOLD, name))
    assert rng0[0] == 0 and 0 < rng0[1] < g["levels_steps"][1]  # both ranks own intervals
    assert it == int(g["iterations"][0]) and conv
    assert gnorm == float(g["g_norm"][0])
    assert np.array_equal(np.asarray(hist), g["history"])
    assert solves == int(g["solves"][0])
    assert mean == float(g["mean_iters"][0])
    assert np.array_equal(traj, g["trajectory"])


def test_partition_covers_intervals():
    for J in (1, 7, 125, 1250):
        for R in range(1, min(J, 9) + 1):
            parts = [TS.partition(J, R, r) for r in range(R)]
            assert parts[0][0] == 0 and parts[-1][1] == J
            assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
            assert max(p[1] - p[0] for p in parts) - min(p[1] - p[0] for p in parts) <= 1
