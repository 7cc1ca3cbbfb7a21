#!/usr/bin/env python
"""Benchmark of the device-resident IPM Newton solve (driver contract).

Headline workload (BASELINE.json configs[4], "C5", the largest configuration
that fits one GPU): 2D heat-equation control, all-at-once backward Euler on
257x257 spatial Q1 nodes x 128 time steps (level 8, tau = 1/128; 33.3M KKT
unknowns), alpha 1e-3, beta 1e-4, u in [-1, 1], seeded sine-mode y_d x
exp(-t), block-diagonal preconditioned MINRES (P_D, the solver BASELINE names
for C5). One step = one IPM solve to tolerance.

metric: Krylov iterations per second over the whole IPM solve (time to
tolerance, per-Newton-step preconditioner setup included). N > 1: replicas,
one solve per rank (SURVEY §8e "replicas only"), scaling "weak", time = max
over ranks. ``--config C2`` runs the previous headline (the 513^2 9-cell
(alpha, beta) sweep), its cells partitioned over the ranks.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config C5|C2]
"""
from __future__ import annotations

import argparse
import ctypes as C
import glob
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "krylov_iters_per_s"
UNIT = "iters/s"
L2_FLUSH_BYTES = 256 << 20
DEFAULT_SOLVER = {"C5": "minres-pd", "C2": "gmres-pt"}
PRECOND_KIND = {"gmres-pt": "pt", "minres-pd": "pd", "gmres-ppi": "ppi"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C5", choices=["C5", "C2"])
    ap.add_argument("--solver", default=None, help="Krylov solver (default: minres-pd for C5, "
                                                   "gmres-pt for C2)")
    ap.add_argument("--smoother", default="auto", choices=["auto", "color4", "lex"])
    ap.add_argument("--level", type=int, default=None, help="override the config's level (testing)")
    ap.add_argument("--nt", type=int, default=None, help="override C5's time steps (testing)")
    ap.add_argument("--replicas", type=int, default=8,
                    help="C5: independent solves in flight per GPU (y_d seeds 42, 43, ...)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the extra measurements (C2 sweep, C3/C4 apply bandwidth)")
    ap.add_argument("--tune", action="append", default=[], help="name=value (oc_set_tuning)")
    a = ap.parse_args()
    a.solver = a.solver or DEFAULT_SOLVER[a.config]
    return a


# ------------------------------------------------------------------ configs
def c5_config(args):
    from paper_1806_05896_b200 import configs

    c = configs.C5
    if args.level is not None or args.nt is not None:
        lvl = args.level or c.level
        nt = args.nt or c.nt
        c = c.with_level(lvl, tau=1.0 / nt)
    return c


def c2_cells(args):
    from paper_1806_05896_b200 import configs

    lvl = args.level or 9
    return [c.with_level(lvl, solver=args.solver) for c in configs.C2_CELLS]


def control_problem(c, y_d=None, u_a=None, u_b=None):
    from paper_1806_05896_b200 import optcon as oc

    kw = dict(pde=c.pde, alpha=c.alpha, beta=c.beta,
              y_d=c.y_d() if y_d is None else y_d,
              u_a=c.u_a if u_a is None else u_a, u_b=c.u_b if u_b is None else u_b)
    if c.pde == "heat":
        kw["tau"] = c.tau
    if c.pde == "convdiff":
        kw["eps"] = c.eps
    if c.y_a is not None:
        kw.update(y_a=c.y_a, y_b=c.y_b)
    if c.obs is not None:
        kw["observation"] = c.obs
    return oc.ControlProblem(**kw)


def workload(args, world=1):
    if args.config == "C5":
        c = c5_config(args)
        nx = (1 << c.level) + 1
        n_kkt = 4 * c.n * c.nt
        return {
            "workload": f"C5: 2D heat-equation control, all-at-once backward Euler, {nx}x{nx} "
                        f"Q1 nodes x {c.nt} time steps (level {c.level}, tau=1/{c.nt}, "
                        f"{n_kkt / 1e6:.1f}M KKT unknowns), {args.solver}, alpha {c.alpha:g}, "
                        f"beta {c.beta:g}, u in [{c.u_a:g},{c.u_b:g}], sigma 0.2, every IPM "
                        "solve to tolerance",
            "level": c.level, "nt": c.nt, "solver": args.solver, "smoother": args.smoother,
            "y_d": "seeded 4 sine modes (seed 42) x exp(-t_k)",
            "replicas_per_gpu": args.replicas,
            "y_d_seeds": c5_seeds(args),
            "parallelism": f"replicas: {args.replicas} independent C5 solves in flight per GPU "
                           "(y_d seeds 42, 43, ...), one per rank-GPU set; no data-path "
                           "collective",
            "l2": "inputs > L2 (67 MB per space-time field); L2 also flushed between steps "
                  "(256 MiB write)",
        }
    lvl = args.level or 9
    return {
        "workload": f"C2: 2D Poisson L1 + control box, {(1 << lvl) + 1}x{(1 << lvl) + 1} nodes "
                    f"(level {lvl}), 9-cell alpha x beta sweep, {args.solver}, sigma 0.2, "
                    "u in [-2,2], every IPM solve to tolerance",
        "level": lvl, "cells": 9, "solver": args.solver, "smoother": args.smoother,
        "alphas": [1e-2, 1e-4, 1e-6], "betas": [1e-2, 1e-3, 1e-4],
        "y_d": "seeded 4 sine modes (seed 42)",
        "parallelism": f"cells partitioned over {world} rank(s), concurrent per GPU",
        "l2": "flushed between steps (256 MiB write)",
    }


# ------------------------------------------------------------ CPU reference
def _ref_problem(c):
    from oracle import ref

    kw = dict(alpha=c.alpha, beta=c.beta, y_d=c.y_d(), u_a=c.u_a, u_b=c.u_b)
    if c.pde == "heat":
        kw["tau"] = c.tau
    if c.pde == "convdiff":
        kw["eps"] = c.eps
    if c.y_a is not None:
        kw.update(y_a=c.y_a, y_b=c.y_b)
    if c.obs is not None:
        kw["obs"] = c.obs
    return ref.RefProblem(c.pde, c.level, **kw)


def c5_ref_sample(args, threads, warm_tasks, timed_tasks):
    """The reference (oracle/_ref: its own assembly, ipm_solve, heat preconditioner
    composition and minres) on the host cores. Each thread owns a replica of
    C5 at its first IPM Newton system (formed by the reference's ipm_solve,
    preconditioner set up once: excluded from the timing, which favours the
    reference); a task = the reference's minres for one iteration on it.
    Tasks are dealt round-robin over the threads and run back to back.
    Returns (iters/s, total iters, wall s, setup s, per-task seconds)."""
    c = c5_config(args)
    solver = "heat-minres-pd" if args.solver == "minres-pd" else "gmres-pt"
    kind, method = ("heat-pd", "minres") if args.solver == "minres-pd" else ("heat-pt", "gmres")
    probs = [None] * threads
    setup = [0.0] * threads
    seeds = c5_seeds(args)

    def prep(i):
        probs[i] = _ref_problem(c.with_level(c.level, seed=seeds[i % len(seeds)]))
        setup[i] = probs[i].newton_sample_prepare(solver)

    _run_threads(prep, range(threads))

    def run_tasks(n_tasks):
        iters, secs = [0] * threads, [[] for _ in range(threads)]

        def work(t):
            for _ in range(t, n_tasks, threads):
                it, _, s = probs[t].newton_sample_run(kind, method, 1)
                iters[t] += it
                secs[t].append(s)

        t0 = time.perf_counter()
        _run_threads(work, range(min(threads, n_tasks)))
        return sum(iters), time.perf_counter() - t0, [s for ss in secs for s in ss]

    run_tasks(warm_tasks)
    it, wall, per = run_tasks(timed_tasks)
    probs.clear()
    return it / wall, it, wall, statistics.mean(setup), per


def c2_ref_sample(args, ipm_iters=2, threads=None):
    """The reference on the host cores: the first `ipm_iters` IPM iterations of
    each C2 cell, one solve per thread."""
    cs = c2_cells(args)
    threads = threads or min(len(cs), os.cpu_count() or 1)
    cs = cs[:threads]
    probs = [_ref_problem(c) for c in cs]
    iters = [0] * len(cs)

    def work(i):
        iters[i] = probs[i].solve(args.solver, sigma=0.2, max_iterations=ipm_iters).total_lin

    t0 = time.perf_counter()
    _run_threads(work, range(len(cs)))
    wall = time.perf_counter() - t0
    return sum(iters) / wall, sum(iters), wall, threads


def _run_threads(fn, idx):
    from paper_1806_05896_b200 import replicas

    replicas.run_concurrent(fn, list(idx))


def ref_cores():
    return os.cpu_count() or 1


def run_reference(args):
    from paper_1806_05896_b200 import replicas

    rank, _, _ = replicas.env_rank()
    if not replicas.reference_runs_on(rank):
        return
    try:
        from oracle import ref

        if not ref.available():
            raise RuntimeError("oracle/_ref/liboptcon_ref.so not built")
        if args.config == "C5":
            # K timed tasks over T threads (T <= cores, equal shares); warm-up:
            # one task per thread that runs timed tasks (first-touch, caches)
            per = -(-args.steps // ref_cores())
            threads = -(-args.steps // per)
            value, it, wall, setup_s, tasks = c5_ref_sample(args, threads, threads, args.steps)
            sample = (f"reference optcon (oracle/_ref: the reference sources compiled -O3, AVX2 "
                      f"kernels) on C5 at full size: {threads} host threads, each with its own "
                      f"replica at the first IPM Newton system (the reference's ipm_solve forms "
                      f"it; its preconditioner set up once, {setup_s:.1f} s, excluded); one step "
                      f"= the reference's {args.solver.split('-')[0]} run for one iteration "
                      f"(mean {statistics.mean(tasks):.1f} s); the {args.steps} timed steps are "
                      f"dealt round-robin over the threads ({per} per thread); warm-up: one "
                      "step per thread")
            cores = threads
            ms_per_step = 1e3 * wall / args.steps
        else:
            for _ in range(args.warmup):
                c2_ref_sample(args)
            tot_it, tot_t = 0, 0.0
            for _ in range(args.steps):
                v, it, wall, cores = c2_ref_sample(args)
                tot_it += it
                tot_t += wall
            value = tot_it / tot_t
            ms_per_step = 1e3 * tot_t / args.steps
            sample = (f"reference optcon (oracle/_ref) first 2 IPM iterations of each of "
                      f"{cores} C2 cells, one solve per thread")
    except Exception as e:  # pragma: no cover - reported, not hidden
        print(json.dumps({"impl": "reference", "unavailable": f"{type(e).__name__}: {e}"}))
        return
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": workload(args), "impl": "reference",
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------- clocks
class ClockSampler:
    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_{os.getpid()}.csv")

    def __enter__(self):
        os.makedirs(os.path.dirname(self.path), exist_ok=True)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.f.close()

    def summary(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        rows = []
        for ln in open(self.path):
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) >= 9:
                rows.append(parts)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        smax = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i] == "Active"})
        loaded = [s for s in sm if smax and s > 0.5 * max(smax)] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(smax) if smax else None, "reasons": reasons,
                "samples": len(rows)}


def measured_peak_hbm():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        return float(json.load(open(p))["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def measured_traffic(kernel):
    """DRAM bytes per launch of the roofline kernel from a committed ncu capture
    (profiles/*/roofline_traffic*.json with a matching "kernel"), or None."""
    best = None
    for f in sorted(glob.glob(os.path.join(ROOT, "profiles", "*", "roofline_traffic*.json"))):
        try:
            d = json.load(open(f))
        except Exception:
            continue
        if d.get("kernel") == kernel:
            best = {"bytes": d["dram_bytes_per_launch"], "source": os.path.relpath(f, ROOT),
                    "blocks_per_launch": d.get("blocks_per_launch", 1)}
    return best


def reference_solve_time(case):
    """The reference's full IPM solve time for a BASELINE case, measured on a
    host of this pool by tools/parity_full.py (profiles/*/parity_full_r*.json),
    with its Newton and average Krylov counts; None when not recorded."""
    best = None
    for f in sorted(glob.glob(os.path.join(ROOT, "profiles", "*", "parity_full_r*.json"))):
        try:
            d = json.load(open(f))
        except Exception:
            continue
        if case in d and "ref_s" in d[case]:
            r = d[case]
            best = {"seconds": r["ref_s"], "nli": r["nli"][1], "av_li": r["av_li"][1],
                    "source": os.path.relpath(f, ROOT)}
    return best


# ------------------------------------------------------------------ ours
def _setup_torch(args):
    import torch

    from paper_1806_05896_b200 import _lib, replicas

    for kv in args.tune:
        k, v = kv.split("=")
        _lib.check(_lib.load().oc_set_tuning(k.encode(), int(v)))
    rank, world, local = replicas.env_rank()
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return torch, dist, rank, world, local


def _barrier(torch, dist):
    if dist:
        dist.barrier()
    torch.cuda.synchronize()


def run_ours(args):
    torch, dist, rank, world, local = _setup_torch(args)
    if args.config == "C5":
        line = run_ours_c5(args, torch, dist, rank, world, local)
    else:
        line = run_ours_c2(args, torch, dist, rank, world, local)
    if rank == 0 and world == 1 and not args.no_extras:
        line["extras"] = run_extras(args, torch, local)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def _pinned_zeros(torch, n):
    return torch.zeros(n, dtype=torch.float64).pin_memory().numpy()


def c5_seeds(args):
    """y_d seeds of the replicas in flight per GPU / host thread (42, 43, ...)."""
    return [42 + i for i in range(args.replicas)]


def run_ours_c5(args, torch, dist, rank, world, local):
    from paper_1806_05896_b200 import bytes_model, configs, optcon as oc, replicas

    c = c5_config(args)
    params = oc.IpmParams(sigma=c.sigma, solver=args.solver, smoother=args.smoother)
    grid = oc.Grid(c.level)
    R = args.replicas
    seeds = c5_seeds(args)
    yds = [configs.sine_modes_spacetime(c.level, c.nt, c.tau, seed=sd) for sd in seeds]
    # one context (CUDA stream) and host thread per replica: the R independent
    # solves overlap on the GPU (each time-block solve occupies one 16-SM cluster)
    ctxs = [oc.Context(local) for _ in range(R)]
    qps = [oc.assemble_spacetime(control_problem(c, y_d=yds[i]), grid, ctxs[i]) for i in range(R)]
    ny = qps[0].ny
    dev = lambda n: torch.empty(n, dtype=torch.float64, device="cuda")  # noqa: E731
    outs = [dict(u=dev(ny), y=dev(ny), z=dev(2 * ny), p=dev(ny), lam_za=dev(2 * ny),
                 lam_zb=dev(2 * ny)) for _ in range(R)]
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device="cuda")

    def solve(i):
        r = oc.ipm_solve(qps[i], params, outputs=outs[i])
        ctxs[i].record(1)
        if not r.stats.converged:
            raise RuntimeError("IPM did not converge in the bench workload")
        return r

    def step():
        for cx in ctxs:
            cx.record(0)
        res = replicas.run_concurrent(solve, range(R))
        ms = max(ctxs[0].elapsed_ms_to(0, ctxs[i], 1) for i in range(R))
        return [res[i] for i in range(R)], ms

    for _ in range(args.warmup):
        step()
    # ---------------------------------------------------------- timed region
    times, iters, results = [], 0, []
    l0 = oc.Context.launch_count()
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.fill_(1.0)  # L2 flush between timed steps (outside the timing)
            _barrier(torch, dist)
            for cx in ctxs:
                cx.synchronize()
            res, ms = step()
            times.append(ms)
            results.append(res)
            _barrier(torch, dist)
            iters += sum(r.total_lin for r in res)
    launches = oc.Context.launch_count() - l0
    max_ms, all_iters = replicas.reduce_step_stats(sum(times), iters, dist, device="cuda")
    value = replicas.aggregate_rate(max_ms, all_iters)

    # ------------------------------------- e2e through the C ABI (host buffers)
    yd_h = [torch.from_numpy(y).pin_memory() for y in yds]
    ua_h = torch.full((c.n,), c.u_a, dtype=torch.float64).pin_memory()
    ub_h = torch.full((c.n,), c.u_b, dtype=torch.float64).pin_memory()
    host_out = [dict(u=_pinned_zeros(torch, ny), y=_pinned_zeros(torch, ny),
                     z=_pinned_zeros(torch, 2 * ny), p=_pinned_zeros(torch, ny)) for _ in range(R)]

    def e2e_one(i):
        q2 = oc.assemble_spacetime(control_problem(c, y_d=yd_h[i].numpy(), u_a=ua_h.numpy(),
                                                   u_b=ub_h.numpy()), grid, ctxs[i])
        r2 = oc.ipm_solve(q2, params, outputs=host_out[i])
        h = q2.h2d_bytes
        q2.close()
        ctxs[i].synchronize()
        return r2.total_lin, h

    e2e_s, e2e_it, h2d = [], 0, 0
    for s in range(max(1, min(args.steps, 2)) + 1):
        _barrier(torch, dist)
        t0 = time.perf_counter()
        res = replicas.run_concurrent(e2e_one, range(R))
        dt = time.perf_counter() - t0
        if s > 0:  # the first pass warms the host-side allocator
            e2e_s.append(dt)
            e2e_it += sum(v[0] for v in res.values())
            h2d = sum(v[1] for v in res.values())
    d2h = sum(8 * a.size for ho in host_out for a in ho.values())
    e2e_max_ms, e2e_all = replicas.reduce_step_stats(1e3 * sum(e2e_s), e2e_it, dist, device="cuda")
    e2e_value = replicas.aggregate_rate(e2e_max_ms, e2e_all)

    # -------- in-situ kernel timing (one untimed step, same R solves in flight):
    # CUDA events around every heat time-block solve (the level-8 cluster
    # kernel) on each replica's solver stream
    flush.fill_(1.0)
    torch.cuda.synchronize()
    for cx in ctxs:
        cx.profile(True)
    t_prof = time.perf_counter()
    replicas.run_concurrent(solve, range(R))
    for cx in ctxs:
        cx.synchronize()
    t_prof = (time.perf_counter() - t_prof) * 1e3
    blk_ms, blk_n = 0.0, 0
    for cx in ctxs:
        pr = cx.profile_read()
        cx.profile(False)
        blk_ms += pr["block"][0]
        blk_n += pr["block"][1]
    peak, peak_src = measured_peak_hbm()
    import ctypes as C
    from paper_1806_05896_b200 import _lib
    chain = C.c_int(0)
    _lib.check(_lib.load().oc_get_tuning(b"heat_chain", C.byref(chain)))
    # one launch = one substitution direction (c.nt chained block solves), or one block solve
    per_launch = c.nt if chain.value else 1
    one_blk_bytes = bytes_model.mg_solve_words(c.level) * 8.0 * c.n
    blk_bytes = one_blk_bytes * per_launch
    kernel = "k_bottom_cluster<8>"
    traffic = measured_traffic(kernel)
    if traffic:
        traffic = dict(traffic, bytes=traffic["bytes"] * per_launch // traffic.get("blocks_per_launch", 1))
    achieved = blk_bytes / (blk_ms / blk_n / 1e3) / 1e9 if blk_n else None
    # one replica alone: IPM time to tolerance and the KKT + P apply bandwidth
    single = solve(0)
    kind = PRECOND_KIND[args.solver]
    kkt_b, prec_b = bytes_model.apply_bytes(kind, c.level, ny, pde="heat")
    kkt_ms, prec_ms = qps[0].time_applies(kind, 3)
    apply_gbs = (kkt_b + prec_b) / ((kkt_ms + prec_ms) / 1e3) / 1e9
    # all replicas together: every KKT + P_D apply of the timed steps (one of each per Krylov
    # iteration plus the P_D apply that starts each Newton solve) over the steps' device time
    n_applies = sum(r.total_lin + r.stats.nli for res in results for r in res)
    agg_gbs = n_applies * (kkt_b + prec_b) / (max_ms / 1e3) / 1e9  # this rank's GPU
    n_chain = n_applies * (2 if per_launch > 1 else 2 * c.nt)  # launches of the block kernel in the timed steps

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            a1 = argparse.Namespace(**vars(args))
            a1.replicas = 1
            v, it, wall, setup_s, per = c5_ref_sample(a1, 1, 0, 1)
            cpu = {"value": v, "unit": UNIT, "cores": 1, "kind": "reference",
                   "sample": f"reference optcon (oracle/_ref) on C5 at full size, 1 thread, "
                             f"seed 42: {it} {args.solver.split('-')[0]} iteration(s) at the first "
                             f"IPM Newton system, {wall:.1f} s (preconditioner setup "
                             f"{setup_s:.1f} s excluded)"}
        except Exception as e:
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                   "sample": f"unavailable: {type(e).__name__}: {e}"}

    ipm_ms = [r.solve_ms for res in results for r in res]
    last = results[-1][0]
    return {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": max_ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded sine-mode y_d x exp(-t); no dataset exists for this path)",
        "config": workload(args, world),
        "roofline": {
            "bound": "hbm", "kernel": f"{kernel} ({per_launch} chained heat time-block multigrid "
                                      "solve(s) per launch, each 3 V-cycles on M + tau L + "
                                      "diag(m_k), 65,025 nodes; one 16-CTA cluster)",
            "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": (achieved / peak) if achieved else None,
            "traffic": traffic["bytes"] if traffic else None,
            "traffic_source": traffic["source"] if traffic else None,
            "peak_source": peak_src, "bytes_per_launch": blk_bytes,
            "avg_launch_ms": blk_ms / blk_n if blk_n else None, "launches_in_pass": blk_n,
            "block_solves_per_launch": per_launch,
            "in_flight": {"launches_in_timed_steps": n_chain,
                          "avg_concurrent_launches": (n_chain * blk_ms / blk_n / max_ms) if blk_n else None,
                          "aggregate_achieved": n_chain * blk_bytes / (max_ms / 1e3) / 1e9,
                          "aggregate_frac": n_chain * blk_bytes / (max_ms / 1e3) / 1e9 / peak,
                          "note": f"the same kernel's launches of all {R} solves in the timed steps "
                                  "(substitution directions x P_D applies) over the steps' device time; at "
                                  "most 7 of these 16-CTA clusters are resident"},
            "avg_block_solve_ms": blk_ms / blk_n / per_launch if blk_n else None,
            "note": "achieved = SURVEY 8d algorithmic bytes of the launch's block MG solves (287 "
                    "words per node each) / its CUDA-event time on the solver streams in an "
                    f"untimed step with the same {R} solves in flight; the kernel is "
                    "latency-bound (256 dependent block solves per preconditioner apply on one "
                    "16-SM cluster, at most 7 such clusters resident; its data stay on chip "
                    "after one read), see DESIGN.md",
        },
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h),
                "what": f"{R} concurrent x (assemble_spacetime from pinned host arrays (upload, "
                        "device setup), ipm_solve, u/y/z/p to pinned host arrays, close); host "
                        "wall clock"},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
        "ipm_time_to_tolerance_ms": {"mean": statistics.mean(ipm_ms), "min": min(ipm_ms),
                                     "max": max(ipm_ms), "note": f"per solve, {R} in flight"},
        "single_solve": {"ipm_time_to_tolerance_ms": single.solve_ms,
                         "krylov_iters_per_s": single.total_lin / (single.solve_ms / 1e3),
                         "nli": single.stats.nli, "av_li": round(single.stats.av_li, 3),
                         "note": "seed 42 alone on the GPU (untimed pass)"},
        "time_to_solution_vs_reference": _tts(single, "C5m" if args.solver == "minres-pd" else "C5"),
        "nli": [r.stats.nli for r in results[-1]], "av_li": [round(r.stats.av_li, 3) for r in results[-1]],
        "lin_iters_seed42": [i.lin_iters for i in last.stats.iterations[1:]],
        "objective_seed42": last.objective,
        "kkt_precond_apply": {"gbs": apply_gbs, "kkt_ms": kkt_ms, "prec_ms": prec_ms,
                              "bytes": kkt_b + prec_b, "frac_of_peak": apply_gbs / peak,
                              "how": "oc_time_applies on replica 0 alone after its last solve "
                                     "(final Theta), CUDA events; SURVEY 8d byte model",
                              "in_flight": {"gbs": agg_gbs, "frac_of_peak": agg_gbs / peak,
                                            "applies": n_applies, "solves_in_flight": R,
                                            "how": "algorithmic bytes of every KKT + P_D apply of "
                                                   "the timed steps (all solves in flight on this "
                                                   "GPU) / the steps' device time, setup and "
                                                   "Krylov vector work included in the time"}},
    }


def _tts(single, case):
    """One solve's IPM time to tolerance against the reference's full solve of
    the same case (one host thread, recorded by tools/parity_full.py): the
    speed-up that counts each side's own Krylov iterations."""
    ref = reference_solve_time(case)
    if not ref:
        return None
    return {"device_s": single.solve_ms / 1e3, "reference_s": ref["seconds"],
            "ratio": ref["seconds"] / (single.solve_ms / 1e3),
            "device_nli_av_li": [single.stats.nli, round(single.stats.av_li, 3)],
            "reference_nli_av_li": [ref["nli"], ref["av_li"]], "reference_source": ref["source"],
            "note": "reference: one host thread of this pool, recorded (not re-run by the bench)"}


def run_ours_c2(args, torch, dist, rank, world, local):
    from paper_1806_05896_b200 import _lib, bytes_model, optcon as oc, replicas

    cs = c2_cells(args)
    mine = replicas.partition(len(cs), rank, world)
    params = oc.IpmParams(sigma=0.2, solver=args.solver, smoother=args.smoother)
    grid = oc.Grid(cs[0].level)
    ctxs = {i: oc.Context(local) for i in mine}
    probs = {i: oc.build_qp(control_problem(cs[i]), grid, ctxs[i]) for i in mine}
    ny = cs[0].n
    dev = lambda n: torch.empty(n, dtype=torch.float64, device="cuda")  # noqa: E731
    outs = {i: dict(u=dev(ny), y=dev(ny), z=dev(2 * ny), p=dev(ny), lam_za=dev(2 * ny),
                    lam_zb=dev(2 * ny)) for i in mine}
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device="cuda")
    c0 = ctxs[mine[0]] if mine else None

    def solve_cell(i):
        r = oc.ipm_solve(probs[i], params, outputs=outs[i])
        if not r.stats.converged:
            raise RuntimeError("IPM did not converge in the bench workload")
        ctxs[i].record(1)
        return r

    def step():
        if not mine:
            return 0, {}, 0.0
        for i in mine:
            ctxs[i].record(0)
        res = replicas.run_concurrent(solve_cell, mine)
        ms = max(c0.elapsed_ms_to(0, ctxs[i], 1) for i in mine)
        return sum(r.total_lin for r in res.values()), res, ms

    for _ in range(args.warmup):
        step()
    times, iters, results = [], 0, {}
    l0 = oc.Context.launch_count()
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.fill_(1.0)
            _barrier(torch, dist)
            for i in mine:
                ctxs[i].synchronize()
            it, results, ms = step()
            times.append(ms)
            _barrier(torch, dist)
            iters += it
    launches = oc.Context.launch_count() - l0
    max_ms, all_iters = replicas.reduce_step_stats(sum(times), iters, dist, device="cuda")
    value = replicas.aggregate_rate(max_ms, all_iters)
    recs = replicas.gather_records(
        {i: dict(nli=r.stats.nli, av_li=round(r.stats.av_li, 3), solve_ms=r.solve_ms,
                 total_lin=r.total_lin, rank=rank) for i, r in results.items()}, len(cs), dist)

    # e2e through the C ABI (pinned host buffers), host wall clock
    pinned = {i: dict(y_d=torch.from_numpy(cs[i].y_d()).pin_memory(),
                      u_a=torch.full((ny,), cs[i].u_a, dtype=torch.float64).pin_memory(),
                      u_b=torch.full((ny,), cs[i].u_b, dtype=torch.float64).pin_memory())
              for i in mine}
    host_out = {i: dict(u=_pinned_zeros(torch, ny), y=_pinned_zeros(torch, ny),
                        z=_pinned_zeros(torch, 2 * ny), p=_pinned_zeros(torch, ny)) for i in mine}

    def e2e_cell(i):
        hp = pinned[i]
        qp = oc.build_qp(control_problem(cs[i], y_d=hp["y_d"].numpy(), u_a=hp["u_a"].numpy(),
                                         u_b=hp["u_b"].numpy()), grid, ctxs[i])
        r = oc.ipm_solve(qp, params, outputs=host_out[i])
        h = qp.h2d_bytes
        qp.close()
        return r.total_lin, h

    e2e_s, e2e_it, h2d = [], 0, 0
    for s in range(max(1, min(args.steps, 2)) + 1):
        _barrier(torch, dist)
        t0 = time.perf_counter()
        res = replicas.run_concurrent(e2e_cell, mine)
        dt = time.perf_counter() - t0
        if s > 0:
            e2e_s.append(dt)
            e2e_it += sum(r[0] for r in res.values())
            h2d = sum(r[1] for r in res.values())
    d2h = sum(8 * a.size for i in mine for a in host_out[i].values())
    e2e_max_ms, e2e_all = replicas.reduce_step_stats(1e3 * sum(e2e_s), e2e_it, dist, device="cuda")
    e2e_value = replicas.aggregate_rate(e2e_max_ms, e2e_all)

    # in-situ timing of the fine-level sweep launches (untimed pass)
    peak, peak_src = measured_peak_hbm()
    sweep_ms, sweep_n = 0.0, 0
    for i in mine:
        ctxs[i].profile(True)
        oc.ipm_solve(probs[i], params, outputs=outs[i])
        pr = ctxs[i].profile_read()
        ctxs[i].profile(False)
        sweep_ms += pr["sweep"][0]
        sweep_n += pr["sweep"][1]
    fuse = C.c_int(0)
    _lib.check(_lib.load().oc_get_tuning(b"sweep_fuse", C.byref(fuse)))
    fuse = max(1, min(5, fuse.value))
    sweep_bytes = fuse * bytes_model.sweep_bytes(ny)
    kernel = f"k_sweep level {cs[0].level} fuse {fuse}"
    traffic = measured_traffic(kernel)
    achieved = sweep_bytes / (sweep_ms / sweep_n / 1e3) / 1e9 if sweep_n else None

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            v, it, wall, cores = c2_ref_sample(args)
            cpu = {"value": v, "unit": UNIT, "cores": cores, "kind": "reference",
                   "sample": f"reference optcon (oracle/_ref) first 2 IPM iterations of each of "
                             f"{cores} C2 cells, one solve per thread"}
        except Exception as e:
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                   "sample": f"unavailable: {type(e).__name__}: {e}"}
    return {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": max_ms / args.steps, "higher_is_better": True,
        "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded sine-mode y_d; no dataset exists for this path)",
        "config": workload(args, world),
        "roofline": {"bound": "hbm", "kernel": kernel, "achieved": achieved, "peak": peak,
                     "unit": "GB/s", "frac": (achieved / peak) if achieved else None,
                     "traffic": traffic["bytes"] if traffic else None,
                     "traffic_source": traffic["source"] if traffic else None,
                     "peak_source": peak_src, "bytes_per_launch": sweep_bytes,
                     "avg_launch_ms": sweep_ms / sweep_n if sweep_n else None},
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h),
                "what": "build_qp from pinned host arrays, ipm_solve, u/y/z/p to pinned host "
                        "arrays, close; this rank's cells concurrent; host wall clock"},
        "gpu_launches": int(launches), "clocks": clk.summary(), "cells": recs,
    }


def run_extras(args, torch, local):
    """Extra measurements next to the headline (N = 1 only): the C2 sweep
    throughput, and the KKT + preconditioner apply bandwidth at the two 1025^2
    configurations (C3 P_Pi, C4 convdiff P_T) on the state after one IPM
    iteration, against the SURVEY 8d byte model."""
    from paper_1806_05896_b200 import bytes_model, configs, optcon as oc

    out = {}
    peak, _ = measured_peak_hbm()
    try:
        ctx = oc.Context(local)
        for name in ("C3", "C4"):
            c = configs.ALL[name]
            qp = oc.build_qp(control_problem(c), oc.Grid(c.level), ctx)
            # colour-sweep smoother: the parallel path (a capped first solve would
            # otherwise switch the auto smoother to the lexicographic sweeps)
            p = oc.IpmParams(sigma=c.sigma, solver=c.solver, max_iterations=1, linear_maxit=3,
                             gmres_restart=c.gmres_restart, smoother="color4")
            try:
                oc.ipm_solve(qp, p)
            except Exception:
                pass  # one capped IPM iteration: only the preconditioner state is used
            kind = PRECOND_KIND[c.solver]
            kkt_ms, prec_ms = qp.time_applies(kind, 20)
            kb, pb = bytes_model.apply_bytes(kind, c.level, qp.ny, pde=c.pde,
                                             state_bounds=c.y_a is not None)
            gbs = (kb + pb) / ((kkt_ms + prec_ms) / 1e3) / 1e9
            out[f"{name}_kkt_precond_apply"] = {
                "kkt_ms": kkt_ms, "prec_ms": prec_ms, "bytes": kb + pb, "gbs": gbs,
                "frac_of_peak": gbs / peak, "kkt_gbs": kb / (kkt_ms / 1e3) / 1e9}
            qp.close()
        ctx.close()
    except Exception as e:
        out["apply_error"] = f"{type(e).__name__}: {e}"
    try:
        a2 = argparse.Namespace(**vars(args))
        a2.config, a2.solver, a2.level, a2.no_cpu_baseline = "C2", "gmres-pt", None, True
        a2.steps, a2.warmup = 3, 2
        line = run_ours_c2(a2, torch, None, 0, 1, local)
        out["C2_sweep"] = {k: line[k] for k in ("value", "unit", "ms_per_step", "e2e")}
        out["C2_sweep"]["roofline_frac"] = line["roofline"]["frac"]
        out["C2_sweep"]["workload"] = line["config"]["workload"]
    except Exception as e:
        out["C2_error"] = f"{type(e).__name__}: {e}"
    return out


def main():
    args = parse()
    from paper_1806_05896_b200 import replicas

    replicas.ensure_world(args.gpus, [os.path.abspath(__file__)] + sys.argv[1:])
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
