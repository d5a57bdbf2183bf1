#!/usr/bin/env python
"""Benchmark: MGRIT time-to-tolerance of the B200 Phi engine (BASELINE.json metric).

One "step" = one full ``MgritSolver::solve()`` (mgrit.hpp:93-118): IC
projection, g-norm solves and MGRIT iterations to the 1e-10 halting
tolerance -- the reference's own timing window (bench.hpp:146-149).  The
metric is DOF*timesteps/s = n_free * Nt / time-to-tol, whole job over all
ranks.

Default workload: BASELINE config 3 (p=4, h=2^-7, Nt=2500, m=4 -- the
reference builds two levels, 2500/625 -- seeded U[-1,1] spline initial
coefficients, f=0), fp64.  Config 4 is the largest config that fits one GPU,
but it is not the default: one C4 solve takes minutes on the B200 and the
reference's own C4 setup alone takes ~25 min on the host (10,001 load
assemblies), so neither arm's 25-step run fits the driver's window; a
single-solve C4 line is committed under profiles/ instead
(`bench.py --config c4 --steps 1 --warmup 0`).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--impl phi|reference]

For N > 1 (torchrun, one rank per GPU) the ONE space-time problem is solved
time-sharded inside the engine (csrc/timeshard.cpp, phi_mgrit_set_comm): each
rank owns a block of the level-0 coarse intervals, halos and the coarse
right-hand sides travel over NCCL, the coarse cycle is replicated -- strong
scaling, identical results for any N.  The reference arm (--impl reference)
runs the unmodified reference (oracle/_ref, compiled from /root/reference)
with all host threads on rank 0; other ranks exit without work.  Configs too
long for the host (C3, C4) are timed on a bounded sample per step:
initialize() + one MGRIT cycle + its residual, extrapolated to the
reference's iteration count (8 at C3).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # BASELINE.json configs[0..3]; two-level where the reference builds two levels
    "c1": dict(p=2, k=4, nt=100, m=4, cycle=2, source_kind=0, source_param=0.0, init_kind=1),
    "c2": dict(p=3, k=6, nt=1000, m=8, cycle=2, source_kind=1, source_param=2 * np.pi ** 2, init_kind=2),
    "c3": dict(p=4, k=7, nt=2500, m=4, cycle=0, source_kind=0, source_param=0.0, init_kind=2),
    "c4": dict(p=5, k=8, nt=10000, m=8, cycle=0, source_kind=1, source_param=2 * np.pi ** 2, init_kind=0),
    # the divisible multilevel variants of C3 / C4 (hard part 2): the
    # reference's build_levels (mgrit.hpp:217-244) gives 3 levels 2560/640/160 with
    # coarse_floor 41, and 4 levels 10240/1280/160/20 with the default floor
    "c3ml": dict(p=4, k=7, nt=2560, m=4, cycle=0, source_kind=0, source_param=0.0, init_kind=2, coarse_floor=41),
    "c4ml": dict(p=5, k=8, nt=10240, m=8, cycle=0, source_kind=1, source_param=2 * np.pi ** 2, init_kind=0),
    # BASELINE.json configs[4]: kernel microbenchmark (SpMV/SpMM and one V(1,1)), p = 2..5, h = 2^-8
    "c5": dict(p=5, k=8, c=1e-4),
}
DEFAULT_CONFIG = "c3"
# the reference's MGRIT iteration count where its full solve is too long for
# the host (SURVEY.md section 6 probes; the engine converges in the same count)
REF_ITERS = {"c3": 8, "c4": 8, "c3ml": 8, "c4ml": 8}
# configs whose reference setup alone is too long for a bench run on the host
HOST_TOO_LONG = {k: ("not run: the reference's setup at h=2^-8, p=5 builds a 10,001-point transient load "
                     "schedule on the host (~25 min, SURVEY.md section 6) and one solve takes ~1.5-2.6 h on "
                     "8 cores; parity at this operator shape is pinned by tests/test_gpu_baseline_parity.py")
                 for k in ("c4", "c4ml")}
FULL_REF_WORK = 5_000_000  # n_free * Nt up to which the reference runs full solves
SEED = 12345


def n_free(cfg):
    return (2 ** cfg["k"] + cfg["p"] - 2) ** 2


def init_coeffs(cfg, rank=0):
    if cfg["init_kind"] != 2:
        return None
    return np.random.default_rng(SEED + rank).uniform(-1.0, 1.0, n_free(cfg))


def workload_name(name, cfg):
    spatial = "Jacobi CG" if cfg.get("spatial_kind") else "p-MG V(1,1) ILUT"
    tag = f"config{name[1]}" + (" multilevel variant" if name.endswith("ml") else "")
    return (f"{tag}: MGRIT p={cfg['p']} h=2^-{cfg['k']} Nt={cfg['nt']} m={cfg['m']} "
            f"{'two-level' if cfg['cycle'] == 2 else 'V-cycle'} FCF, {spatial}, fp64")


def level_steps(cfg):
    """The reference's time-grid hierarchy (build_levels, mgrit.hpp:217-244)."""
    m, steps = cfg["m"], [cfg["nt"]]
    while steps[-1] % m == 0 and steps[-1] >= m:
        nxt = steps[-1] // m
        if len(steps) > 1 and nxt + 1 <= cfg.get("coarse_floor", 8):
            break
        steps.append(nxt)
        if cfg["cycle"] == 2:
            break
    return steps


def shared_config(name, cfg):
    """The `config` object both arms print (identical keys and values)."""
    return {"workload": workload_name(name, cfg), "n_free": n_free(cfg), "Nt": cfg["nt"], "m": cfg["m"],
            "levels": level_steps(cfg),
            "l2": "flushed between timed steps (256 MB read); operators and state are re-read from HBM"}


def full_reference(cfg):
    return cfg["nt"] * n_free(cfg) <= FULL_REF_WORK


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            f = [x.strip() for x in line.split(",")]
            if len(f) < 6:
                continue
            try:
                sm.append(float(f[0]))
                smax = float(f[1])
            except ValueError:
                continue
            for nm, v in zip(names, f[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def allreduce_max(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def allreduce_sum(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


# ---------------------------------------------------------------------------
# CPU legs (reference compiled from /root/reference; oracle restatement as fallback)
# ---------------------------------------------------------------------------
def ref_solver(cfg, workers):
    from oracle import oracle as O
    return O.RefMgrit(cfg["p"], cfg["k"], cfg["nt"], source_kind=cfg["source_kind"],
                      source_param=cfg["source_param"], init_kind=cfg["init_kind"],
                      init_coeffs=init_coeffs(cfg), cycle=cfg["cycle"], m=cfg["m"], workers=workers,
                      coarse_floor=cfg.get("coarse_floor", 8), spatial_kind=cfg.get("spatial_kind", 0))


def ref_step(rm, cfg, name):
    """One reference step: a full solve() where the host finishes it in
    seconds, else initialize() + 1 cycle + residual extrapolated to the
    reference's iteration count.  Returns (seconds, sample text, details)."""
    if full_reference(cfg):
        r = rm.solve()
        return r["wall"], f"full MGRIT solve() ({r['iterations']} iterations)", r
    t_init, t_cyc, hist = rm.partial(1)
    iters = REF_ITERS.get(name, 8)
    return (t_init + iters * t_cyc,
            f"initialize() {t_init:.2f} s + 1 MGRIT cycle with its residual {t_cyc:.2f} s, "
            f"extrapolated to the reference's {iters} iterations", {"hist": hist})


def cpu_baseline_and_parity(cfg, name, sol, res_eng):
    """The reference on the box's host cores (cpu_baseline) and, on the same
    run, the parity of the benchmarked engine mode against it.  Full-solve
    configs compare the whole solve; the others compare the state after one
    MGRIT iteration from initialize(), with per-solve p-MG counts of the
    residual wave."""
    from oracle import oracle as O
    cores = os.cpu_count() or 1
    if not O.ref_available():
        return ({"value": None, "unit": "DOF*timesteps/s", "cores": cores, "kind": "reference",
                 "sample": "unavailable: oracle/_ref not built"}, None)
    n, nt = n_free(cfg), cfg["nt"]
    if name in HOST_TOO_LONG:
        return ({"value": None, "unit": "DOF*timesteps/s", "cores": cores, "kind": "reference",
                 "sample": HOST_TOO_LONG[name]}, None)
    rm = ref_solver(cfg, cores)
    wall, sample, det = ref_step(rm, cfg, name)
    base = {"value": n * nt / wall, "unit": "DOF*timesteps/s", "cores": cores, "kind": "reference",
            "sample": sample + f", workers={cores}", "seconds": wall}

    def rel(a, b):
        return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))

    if full_reference(cfg):
        par = {"compared": "full solve() on identical inputs",
               "mgrit_iterations": [res_eng.iterations, det["iterations"]],
               "spatial_solves": [res_eng.total_spatial_solves, det["total_spatial_solves"]],
               "mean_spatial_iterations": [res_eng.mean_spatial_iterations, det["mean_spatial_iterations"]],
               "final_relative_residual": [res_eng.final_relative_residual, det["final_relative_residual"]],
               "rel_l2_vs_ref": rel(sol.trajectory(), rm.trajectory())}
    else:
        g = sol.initialize()
        sol.mgrit_cycle(0)
        it_e = sol.residual_iters(0)
        r_e = sol.residual_norm(0) / (g if g > 0 else 1.0)
        it_r = rm.residual_iters(0, cores)
        d = np.abs(it_e.astype(np.int64) - it_r.astype(np.int64))
        ue = sol.trajectory()
        ur = np.concatenate([rm.points(0, 0, k0, min(500, nt + 1 - k0)) for k0 in range(0, nt + 1, 500)])
        par = {"compared": "state after initialize() + 1 MGRIT iteration, identical inputs",
               "relative_residual_after_1": [r_e, float(det["hist"][0])],
               "rel_l2_vs_ref": rel(ue, ur),
               "per_solve_pmg_cycles": {"solves": int(nt), "max_abs_diff": int(d.max()),
                                        "differing": int((d > 0).sum())},
               "mgrit_iterations_full_solve": [res_eng.iterations, REF_ITERS.get(name)]}
    par["bar"] = "iteration counts +-1, space-time rel L2 <= 1e-8 (north star)"
    return base, par


REF_BUDGET_S = 300


def run_reference(args, cfg, name):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    cores = os.cpu_count() or 1
    from oracle import oracle as O
    if not O.ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libmiga_ref.so not built"}))
        return
    n, nt = n_free(cfg), cfg["nt"]
    if name in HOST_TOO_LONG:
        print(json.dumps({"impl": "reference", "unavailable": HOST_TOO_LONG[name]}))
        return
    rm = ref_solver(cfg, cores)
    for _ in range(args.warmup):
        rm.initialize()  # warm the thread pool and caches; bounded
    # each step is one bounded sample (ref_step); the whole run is kept to a few
    # minutes: past REF_BUDGET_S of sampling (and at least 3 samples) the remaining
    # steps are not run, and the line says how many were
    times, sample, t_begin = [], "", time.perf_counter()
    for _ in range(args.steps):
        t, sample, _ = ref_step(rm, cfg, name)
        times.append(t)
        if len(times) >= 3 and time.perf_counter() - t_begin > REF_BUDGET_S:
            break
    if len(times) < args.steps:
        sample += f"; {len(times)} of {args.steps} samples run ({REF_BUDGET_S} s sampling budget)"
    t = float(np.mean(times))
    v = n * nt / t
    line = {"metric": "MGRIT time-to-tol, DOF*timesteps/s", "value": v, "unit": "DOF*timesteps/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3,
            "higher_is_better": True, "scaling": "strong", "impl": "reference", "dtype": "f64",
            "data": "synthetic (seeded U[-1,1] spline coefficients, analytic source)",
            "config": shared_config(name, cfg), "vs_baseline": None,
            "run": {"parallelism": f"{cores} CPU threads (MgritConfig::workers)", "sample": sample},
            "cpu_baseline": {"value": v, "unit": "DOF*timesteps/s", "cores": cores, "kind": "reference",
                             "sample": sample},
            "e2e": {"value": v, "unit": "DOF*timesteps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
def c5_traffic():
    """DRAM bytes of the captured p=5 SpMV launch (profiles/traffic.json), or None."""
    try:
        return json.load(open(os.path.join(ROOT, "profiles", "traffic.json"))).get("c5")
    except Exception:
        return None


def run_c5(args, cfg):
    """BASELINE config 5: A x for B in {1, 16, 64} right-hand sides (SpMV / SpMM
    of A = M + 1e-4 K, p = 2..5, h = 2^-8) and one V(1,1) cycle from x0 = 0,
    device-timed (CUDA events), L2 flushed between repetitions.  Algorithmic
    bytes per SURVEY 8(d): SpMM 8 nnz(A) + 16 B n; V-cycle: matrix part
    (wave_report's per-cycle model) + 37 x 8 B n per right-hand side."""
    import paper_2107_05337_b200 as P
    from paper_2107_05337_b200.engine import lib
    rank, world, local = dist_env()
    if rank != 0:
        return
    lib().phi_set_device(local)
    peak, peak_kind = peaks()
    rows = []
    clocks = ClockSampler(local)
    clocks.start()
    for p in (2, 3, 4, 5):
        d = P.SpatialDiscretization.build(p, cfg["k"])
        h = P.PMultigridHierarchy(d, cfg["c"])
        n = d.n_free
        side = int(round(n ** 0.5))
        nnz = (side * (2 * p + 1) - p * (p + 1)) ** 2
        for b in (1, 16, 64):
            # average launch duration over back-to-back launches cycling through four
            # copies of the operator (> L2 in total); "single": L2 flushed by a read,
            # events around one launch (carries the event pair and the idle start,
            # ~4 us of a ~10-20 us kernel: a plain read of the same bytes reaches
            # 62 % of the measured peak that way at p = 5, 26 % at p = 2)
            ms = h.time_kernel(0, b, reps=max(5, args.steps), flush_l2=2)
            ms1 = h.time_kernel(0, b, reps=max(3, args.steps), flush_l2=1)
            by = 8 * nnz + b * 16 * n
            rows.append({"p": p, "B": b, "kernel": "spmm", "us": ms * 1e3, "alg_MB": by / 1e6,
                         "GBs": by / ms / 1e6, "frac": by / ms / 1e6 / peak,
                         "us_single": ms1 * 1e3, "frac_single": by / ms1 / 1e6 / peak})
        for b in (1, 16, 64):
            ms = h.time_kernel(1, b, reps=max(2, args.steps))
            by = h.vcycle_bytes(b)  # SURVEY 8(d) model: operators once per batch + 8 B per vector entry per RHS
            rows.append({"p": p, "B": b, "kernel": "vcycle", "us": ms * 1e3, "alg_MB": by / 1e6,
                         "GBs": by / ms / 1e6, "frac": by / ms / 1e6 / peak, "cycles_per_s": b / (ms * 1e-3)})
    clk = clocks.stop()
    for r in rows:  # SpMM flops (2 per stored nonzero and right-hand side): past the FP64 ridge at large B
        if r["kernel"] == "spmm":
            side = 2 ** cfg["k"] + r["p"] - 2
            nnz = (side * (2 * r["p"] + 1) - r["p"] * (r["p"] + 1)) ** 2
            r["fp64_TFLOPs"] = 2.0 * nnz * r["B"] / (r["us"] * 1e-6) / 1e12
    spmm5 = [r for r in rows if r["kernel"] == "spmm" and r["p"] == 5 and r["B"] == 1][0]
    line = {"metric": "SpMV/SpMM HBM GB/s (config 5 kernel microbenchmark)", "value": spmm5["GBs"], "unit": "GB/s",
            "n_gpus": 1, "steps": args.steps, "warmup": 1, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded N(0,1) right-hand sides)",
            "config": {"workload": "config5: A x and one V(1,1) on A = M + 1e-4 K, p=2..5, h=2^-8, B in {1,16,64}",
                       "l2": "SpMV/SpMM: inputs larger than L2 (launches cycle through four copies of the tiled "
                             "operator, 4 x 64 MB at p=5), 'us_single': flushed by a 256 MB read before each launch; "
                             "V-cycle: flushed between repetitions (256 MB read: clean lines, no write-backs)"},
            "roofline": {"kernel": "spmv_tma_kernel (p=5, B=1)", "bound": "hbm", "achieved": spmm5["GBs"], "peak": peak,
                         "peak_kind": peak_kind, "unit": "GB/s", "frac": spmm5["frac"], "traffic": c5_traffic()},
            "clocks": clk, "table": rows}
    print(json.dumps(line), flush=True)


def run_partial(args, cfg, name):
    """Large configs (C4): initialize() + one MGRIT cycle and residual, timed on
    the device and extrapolated to the reference probe's 8 iterations (the same
    sample as the CPU leg)."""
    import torch
    import paper_2107_05337_b200 as P
    from paper_2107_05337_b200.engine import lib
    rank, world, local = dist_env()
    if rank != 0:
        return
    torch.cuda.set_device(local)
    lib().phi_set_device(local)
    n, nt = n_free(cfg), cfg["nt"]
    disc = P.SpatialDiscretization.build(cfg["p"], cfg["k"])
    sol = P.MgritSolver(disc, nt, source_kind=cfg["source_kind"], source_param=cfg["source_param"],
                        init_kind=cfg["init_kind"], init_coeffs=init_coeffs(cfg), cycle=cfg["cycle"], m=cfg["m"])

    def timed(fn):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        out = fn()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / 1e3, out

    clocks = ClockSampler(local)
    clocks.start()
    t_init, g = timed(sol.initialize)
    t_cyc, _ = timed(lambda: (sol.mgrit_cycle(0), sol.residual_norm(0)))
    clk = clocks.stop()
    iters = 8
    t = t_init + iters * t_cyc
    line = {"metric": "MGRIT time-to-tol, DOF*timesteps/s", "value": n * nt / t, "unit": "DOF*timesteps/s",
            "n_gpus": 1, "steps": 1, "warmup": 0, "ms_per_step": t * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (analytic source, zero initial state)",
            "config": {"workload": workload_name(name, cfg), "n_free": n, "Nt": nt,
                       "sample": f"initialize() {t_init:.2f} s + 1 MGRIT cycle + residual {t_cyc:.2f} s, "
                                 f"extrapolated to {iters} iterations (the reference probe's count)"},
            "clocks": clk}
    print(json.dumps(line), flush=True)


def run_phi(args, cfg, name):
    rank, world, local = dist_env()
    import torch
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    import paper_2107_05337_b200 as P
    from paper_2107_05337_b200.engine import lib
    if torch.cuda.is_available():
        torch.cuda.set_device(local)
    lib().phi_set_device(local)

    n, nt = n_free(cfg), cfg["nt"]
    coeffs = init_coeffs(cfg)
    disc = P.SpatialDiscretization.build(cfg["p"], cfg["k"])
    from paper_2107_05337_b200.engine import default_solver_config
    sol = P.MgritSolver(disc, nt, source_kind=cfg["source_kind"], source_param=cfg["source_param"],
                        init_kind=cfg["init_kind"], init_coeffs=coeffs, cycle=cfg["cycle"], m=cfg["m"],
                        coarse_floor=cfg.get("coarse_floor", 8),
                        solver=default_solver_config(kind=cfg.get("spatial_kind", 0)))
    if world > 1:  # one problem, level 0 sharded over the ranks inside the engine (C++ + NCCL)
        from paper_2107_05337_b200 import timeshard as TS
        comm = TS.nccl_comm_from_torch()
        sol.set_comm(comm)
    solve_fn = sol.solve

    def timed(fn):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        s.record()
        out = fn()
        e.record()
        torch.cuda.synchronize()
        return s.elapsed_time(e) / 1e3, out

    for _ in range(args.warmup):
        res = solve_fn()

    # L2 flush between timed steps, outside the timed region: a read of 256 MB
    # (> the 126 MB L2), leaving clean lines (a write would leave the timed
    # step the write-backs)
    flush_buf = torch.zeros(32 * 1024 * 1024, dtype=torch.float64, device="cuda")

    # ---- device-resident timed region (value)
    clocks = ClockSampler(local)
    barrier(world)
    torch.cuda.synchronize()
    clocks.start()
    times, launches = [], 0
    for _ in range(args.steps):
        flush_buf.sum()
        torch.cuda.synchronize()
        t, res = timed(solve_fn)
        times.append(t)
        launches += sol.launches()  # solve() resets the counter
    clk = clocks.stop()
    barrier(world)
    t_step = allreduce_max(float(np.mean(times)), world)
    value = n * nt / t_step  # one problem (world 1) or one problem sharded over the ranks

    # ---- end to end through the public API with host buffers
    e2e_steps = max(1, min(args.steps, 2))
    pinned_in = torch.empty(n, dtype=torch.float64).pin_memory() if coeffs is not None else None
    pinned_out = torch.empty((nt + 1) * n, dtype=torch.float64).pin_memory()
    from paper_2107_05337_b200.engine import _check, _p
    import ctypes as C

    def e2e_step():
        if pinned_in is not None:
            pinned_in.numpy()[:] = coeffs
            sol._coeffs = pinned_in.numpy()
            _check(lib().phi_mgrit_set_init_coeffs(sol.h, C.c_void_p(pinned_in.data_ptr())))
        r = sol.solve()
        _check(lib().phi_mgrit_trajectory(sol.h, C.c_void_p(pinned_out.data_ptr())))  # gathers when sharded
        return r

    barrier(world)
    e2e_t = []
    for _ in range(e2e_steps):
        t0 = time.perf_counter()
        e2e_step()
        e2e_t.append(time.perf_counter() - t0)
    t_e2e = allreduce_max(float(np.mean(e2e_t)), world)
    e2e = {"value": n * nt / t_e2e, "unit": "DOF*timesteps/s",
           "h2d_bytes_per_step": int(8 * n if coeffs is not None else 0),
           "d2h_bytes_per_step": int(8 * n * (nt + 1)), "ms_per_step": t_e2e * 1e3}

    # ---- roofline of the dominant kernel (phi_wave_kernel), profiled solve
    sol.set_profile(True)
    sol.solve()
    per_level = sol.wave_levels()
    n_waves, wave_ms, wave_bytes = sol.wave_report()
    sol.set_profile(False)
    peak, peak_kind = peaks()
    # side-stream waves run beside the coarse march, so the summed launch durations can
    # exceed the step: the kernel's busy time is then the step itself
    busy_ms = min(wave_ms, t_step * 1e3) if wave_ms > 0 else 0.0
    achieved = wave_bytes / (busy_ms * 1e-3) / 1e9 if busy_ms > 0 else 0.0
    traffic = traffic_note = traffic_alg = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            key = name + ("_cg" if cfg.get("spatial_kind") else "")
            tj = json.load(open(tpath))
            traffic = tj.get(key)  # DRAM bytes of one captured wave launch
            traffic_note = tj.get("_note_" + key) or tj.get("_note")
            traffic_alg = tj.get(key + "_algorithmic")
        except Exception:
            traffic = None
    # Latency model of the same kernel: the solve is a chain of dependent
    # steps (ILUT blocks, Gauss-Seidel lines), so its bound is cycles per
    # dependent step, not bandwidth.  The coarsest level runs one right-hand
    # side at a time (the serial march, mgrit.hpp:188-194): its time per
    # p-MG cycle over the steps of one V-cycle's chain.
    coarse = per_level[-1]
    f_mhz = clk.get("sm_mhz") or 1965.0
    latency = None
    if coarse["cycles"] > 0 and coarse["chain_steps"] > 0:
        ms_cycle = coarse["ms"] / coarse["cycles"]
        latency = {"level": coarse["level"], "serial_phi_solves": coarse["solves"],
                   "pmg_cycles": coarse["cycles"], "ms_per_pmg_cycle": ms_cycle,
                   "dependent_steps_per_vcycle": coarse["chain_steps"],
                   "cycles_per_dependent_step": ms_cycle * 1e-3 * f_mhz * 1e6 / coarse["chain_steps"],
                   "share_of_kernel_time": coarse["ms"] / wave_ms if wave_ms > 0 else None,
                   "note": "per-cycle time includes the residual checks and the right-hand-side product"}
    roofline = {"kernel": "phi_wave_kernel (fused batched Phi solve)", "bound": "hbm", "achieved": achieved,
                "peak": peak, "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic, "traffic_launch": traffic_note, "traffic_launch_algorithmic": traffic_alg,
                "waves": n_waves, "kernel_ms_per_step": wave_ms, "kernel_busy_ms_per_step": busy_ms,
                "algorithmic_bytes_per_step": wave_bytes,
                "per_level": per_level, "latency": latency,
                "note": ("latency-bound, not bandwidth-bound: the serial coarse march runs ILUT block "
                         "recurrences and Gauss-Seidel line scans as dependent chains; 'latency' gives "
                         "the cycles per dependent step that explain the time"
                         if not cfg.get("spatial_kind") else
                         "CG: one SpMV and three dot products per iteration, L2-resident operator")}

    launches = int(allreduce_sum(float(launches), world))  # all ranks' kernels
    line = {"metric": "MGRIT time-to-tol, DOF*timesteps/s", "value": value, "unit": "DOF*timesteps/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_step * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded U[-1,1] spline coefficients, analytic source)",
            "config": shared_config(name, cfg),
            "run": {"mgrit_iterations": res.iterations, "spatial_solves": res.total_spatial_solves,
                    "mean_spatial_iterations": res.mean_spatial_iterations,
                    "parallelism": ("single GPU" if world == 1 else
                                    f"MGRIT level 0 time-sharded over {world} GPUs in the engine (NCCL halo "
                                    f"shifts + allgathered coarse rhs; coarse cycle replicated)"),
                    "summation": "reassociated (default; within north-star tolerance)"},
            "e2e": e2e, "roofline": roofline, "gpu_launches": launches, "clocks": clk}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"], line["parity"] = cpu_baseline_and_parity(cfg, name, sol, res)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=int(os.environ.get("WORLD_SIZE", 1)))
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="phi", choices=["phi", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--partial", action="store_true",
                    help="initialize + one cycle, extrapolated (large configs)")
    ap.add_argument("--solver", default="pmg", choices=["pmg", "cg"],
                    help="spatial solver of Phi (SpatialSolverKind, theta.hpp:64); the headline is pmg")
    args = ap.parse_args()
    cfg = dict(CONFIGS[args.config])
    cfg["spatial_kind"] = 1 if args.solver == "cg" else 0
    if args.config == "c5":
        if args.impl == "reference":
            print(json.dumps({"impl": "reference", "unavailable": "config 5 is a GPU kernel microbenchmark"}))
        else:
            run_c5(args, cfg)
    elif args.impl == "reference":
        run_reference(args, cfg, args.config)
    elif args.partial:
        run_partial(args, cfg, args.config)
    else:
        run_phi(args, cfg, args.config)


if __name__ == "__main__":
    main()
