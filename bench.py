#!/usr/bin/env python
"""Benchmark of the device-resident IPM Newton solve (driver contract).

Workload (BASELINE.json configs[1], "C2"): 2D Poisson L1 + control-box problem
at 513x513 nodes (level 9), the 9-cell sweep alpha in {1e-2,1e-4,1e-6} x beta
in {1e-2,1e-3,1e-4}, seeded sine-mode y_d, block-triangular preconditioned
GMRES (the reference default). One step = the 9 IPM solves to tolerance.

metric: Krylov iterations per second over whole IPM solves (time-to-tolerance
of every cell, setup included). N > 1: independent replicas of the sweep per
rank (SURVEY §8e "replicas only"), scaling "weak", time = max over ranks.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import ctypes as C
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


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--level", type=int, default=9)
    ap.add_argument("--solver", default="gmres-pt")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--sweep-fuse", type=int, default=None,
                    help="smoothing sweeps fused per tiled launch (1..5; library default if unset)")
    ap.add_argument("--sweep-tile", type=int, default=None, help="tiled sweep shape id (tuning)")
    ap.add_argument("--cluster-bottom", type=int, default=None,
                    help="1: levels <= 7 in the 16-CTA cluster kernel (default), 0: tiled + single CTA")
    return ap.parse_args()


def cells(level, solver):
    from paper_1806_05896_b200 import configs

    return [c.with_level(level, solver=solver) for c in configs.C2_CELLS]


def workload(level, solver):
    return {
        "workload": f"C2: 2D Poisson L1 + control box, {(1 << level) + 1}x{(1 << level) + 1} nodes "
                    f"(level {level}), 9-cell alpha x beta sweep, {solver}, sigma 0.2, "
                    "u in [-2,2], every IPM solve to tolerance",
        "level": level, "cells": 9, "solver": solver, "alphas": [1e-2, 1e-4, 1e-6],
        "betas": [1e-2, 1e-3, 1e-4], "y_d": "seeded 4 sine modes (seed 42)",
        "parallelism": "replicas", "l2": "flushed between steps (256 MiB write)",
    }


# ------------------------------------------------------------ CPU baseline
def cpu_reference_sample(level, solver, ipm_iters=2, threads=None):
    """The reference CPU implementation (oracle/_ref) on the host cores: the
    first `ipm_iters` IPM iterations of each C2 cell, one solve per thread.
    Returns (iters_per_s, cores, kind, sample, total_iters, wall_s)."""
    from oracle import ref

    cs = cells(level, solver)
    threads = threads or min(len(cs), os.cpu_count() or 1)
    cs = cs[:threads]  # one cell per host thread: no straggler round
    if ref.available():
        probs = [ref.RefProblem("poisson", c.level, alpha=c.alpha, beta=c.beta, y_d=c.y_d(),
                                u_a=c.u_a, u_b=c.u_b) for c in cs]
        iters = [0] * len(cs)

        def work(i):
            r = probs[i].solve(solver, sigma=0.2, max_iterations=ipm_iters)
            iters[i] = r.total_lin

        t0 = time.perf_counter()
        pool = []
        nxt = [0]
        lock = threading.Lock()

        def runner():
            while True:
                with lock:
                    i = nxt[0]
                    nxt[0] += 1
                if i >= len(cs):
                    return
                work(i)

        for _ in range(threads):
            th = threading.Thread(target=runner)
            th.start()
            pool.append(th)
        for th in pool:
            th.join()
        wall = time.perf_counter() - t0
        sample = (f"reference optcon (oracle/_ref, -O3 AVX2) first {ipm_iters} IPM iterations of "
                  f"each of {len(cs)} C2 cells (level {level}, {solver}), {threads} threads, one solve "
                  "per thread")
        return sum(iters) / wall, threads, "reference", sample, sum(iters), wall
    # fallback: the numpy restatement, one IPM iteration of one cell, 1 thread
    from oracle import port

    c = cs[0]
    qp = port.Qp(level=level, pde="poisson", alpha=c.alpha, beta=c.beta, y_d=c.y_d(), u_a=c.u_a,
                 u_b=c.u_b)
    t0 = time.perf_counter()
    r = port.ipm_solve(qp, sigma=0.2, solver=solver, max_newton=1)
    wall = time.perf_counter() - t0
    sample = f"numpy port, first IPM iteration of one C2 cell (level {level}), 1 thread"
    return r["total_lin"] / wall, 1, "port", sample, r["total_lin"], wall


def run_reference(args):
    from paper_1806_05896_b200 import replicas

    rank, _, _ = replicas.env_rank()
    if not replicas.reference_runs_on(rank):
        return
    try:
        for _ in range(args.warmup):
            cpu_reference_sample(args.level, args.solver)
        tot_it, tot_t = 0, 0.0
        for _ in range(args.steps):
            v, cores, kind, sample, it, wall = cpu_reference_sample(args.level, args.solver)
            tot_it += it
            tot_t += wall
    except Exception as e:  # pragma: no cover - reported, not hidden
        print(json.dumps({"impl": "reference", "unavailable": f"{type(e).__name__}: {e}"}))
        return
    value = tot_it / tot_t
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot_t / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": workload(args.level, args.solver), "impl": "reference",
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind,
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


# ------------------------------------------------------------------ ours
def measured_traffic(level, fuse):
    """DRAM bytes per launch of the roofline kernel from a committed ncu capture
    (profiles/*/roofline_traffic.json), or None."""
    import glob

    best = None
    for f in sorted(glob.glob(os.path.join(os.path.dirname(os.path.abspath(__file__)),
                                           "profiles", "*", "roofline_traffic.json"))):
        try:
            d = json.load(open(f))
        except Exception:
            continue
        if d.get("level") == level and d.get("fuse") == fuse:
            best = {"bytes": d["dram_bytes_per_launch"], "source": os.path.relpath(f)}
    return best


def run_ours(args):
    import torch

    from paper_1806_05896_b200 import _lib, bytes_model, optcon as oc, replicas

    if args.sweep_fuse is not None:
        _lib.check(_lib.load().oc_set_tuning(b"sweep_fuse", int(args.sweep_fuse)))
    if args.sweep_tile is not None:
        _lib.check(_lib.load().oc_set_tuning(b"sweep_tile", int(args.sweep_tile)))
    if args.cluster_bottom is not None:
        _lib.check(_lib.load().oc_set_tuning(b"cluster_bottom", int(args.cluster_bottom)))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        if dist:
            dist.barrier()
        torch.cuda.synchronize()

    cs = cells(args.level, args.solver)
    params = oc.IpmParams(sigma=0.2, solver=args.solver)
    grid = oc.Grid(args.level)
    # one context (CUDA stream) per cell: the 9 independent solves of the sweep run
    # concurrently on the GPU, as the reference's run_sweep runs them on a thread pool
    ctxs = [oc.Context(local) for _ in cs]
    probs = [oc.build_qp(oc.ControlProblem(alpha=c.alpha, beta=c.beta, y_d=c.y_d(), u_a=c.u_a,
                                           u_b=c.u_b), grid, cx) for c, cx in zip(cs, ctxs)]
    ny = probs[0].ny
    outs = [dict(u=torch.empty(ny, dtype=torch.float64, device="cuda"),
                 y=torch.empty(ny, dtype=torch.float64, device="cuda"),
                 z=torch.empty(2 * ny, dtype=torch.float64, device="cuda"),
                 p=torch.empty(ny, dtype=torch.float64, device="cuda"),
                 lam_za=torch.empty(2 * ny, dtype=torch.float64, device="cuda"),
                 lam_zb=torch.empty(2 * ny, dtype=torch.float64, device="cuda")) for _ in cs]
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device="cuda")

    def run_concurrent(fn):
        """fn(i) for every cell on its own host thread; returns results in cell order."""
        res = [None] * len(cs)
        err = []

        def body(i):
            try:
                res[i] = fn(i)
            except Exception as e:  # re-raised on the main thread
                err.append(e)

        th = [threading.Thread(target=body, args=(i,)) for i in range(len(cs))]
        for t in th:
            t.start()
        for t in th:
            t.join()
        if err:
            raise err[0]
        return res

    def solve_cell(i):
        r = oc.ipm_solve(probs[i], params, outputs=outs[i])
        if not r.stats.converged:
            raise RuntimeError("IPM did not converge in the bench workload")
        ctxs[i].record(1)
        return r

    def step():
        for cx in ctxs:
            cx.record(0)
        res = run_concurrent(solve_cell)
        ms = max(ctxs[0].elapsed_ms_to(0, cx, 1) for cx in ctxs)
        return sum(r.total_lin for r in res), res, ms

    for _ in range(args.warmup):
        step()
    # ---------------------------------------------------------- timed region
    times, iters, results = [], 0, None
    l0 = oc.Context.launch_count()
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.fill_(1.0)           # L2 flush between timed steps (outside timing)
            barrier()
            for cx in ctxs:
                cx.synchronize()
            it, results, ms = step()
            times.append(ms)
            barrier()
            iters += it
    launches = oc.Context.launch_count() - l0
    total_ms = sum(times)
    max_ms, all_iters = replicas.reduce_step_stats(total_ms, iters, dist, device="cuda")
    value = replicas.aggregate_rate(max_ms, all_iters)

    # ------------------------------------------- e2e through the C ABI (host buffers)
    pinned = [dict(y_d=torch.from_numpy(c.y_d()).pin_memory(),
                   u_a=torch.full((ny,), c.u_a, dtype=torch.float64).pin_memory(),
                   u_b=torch.full((ny,), c.u_b, dtype=torch.float64).pin_memory()) for c in cs]
    def pinned_zeros(n):
        return torch.zeros(n, dtype=torch.float64).pin_memory().numpy()

    host_out = [dict(u=pinned_zeros(ny), y=pinned_zeros(ny), z=pinned_zeros(2 * ny),
                     p=pinned_zeros(ny)) for _ in cs]

    def e2e_cell(i):
        c, hp = cs[i], pinned[i]
        qp = oc.build_qp(oc.ControlProblem(alpha=c.alpha, beta=c.beta, y_d=hp["y_d"].numpy(),
                                           u_a=hp["u_a"].numpy(), u_b=hp["u_b"].numpy()),
                         grid, ctxs[i])
        r = oc.ipm_solve(qp, params, outputs=host_out[i])
        ctxs[i].record(3)
        h = qp.h2d_bytes
        qp.close()
        return r.total_lin, h

    e2e_ms, e2e_it, h2d = [], 0, 0
    for s in range(max(1, min(args.steps, 2)) + 1):
        barrier()
        for cx in ctxs:
            cx.synchronize()
            cx.record(2)
        res = run_concurrent(e2e_cell)
        dt_ms = max(ctxs[0].elapsed_ms_to(2, cx, 3) for cx in ctxs)
        if s > 0:  # first pass warms the host-side allocator
            e2e_ms.append(dt_ms)
            e2e_it += sum(r[0] for r in res)
            h2d = sum(r[1] for r in res)
    d2h = sum(8 * (a.size) for a in host_out[0].values()) * len(cs)
    e2e_max_ms, e2e_all_it = replicas.reduce_step_stats(sum(e2e_ms), e2e_it, dist, device="cuda")
    e2e_value = replicas.aggregate_rate(e2e_max_ms, e2e_all_it)

    # ---- in-situ kernel timing pass (untimed; cells one at a time, events per launch)
    prof = {"sweep": [0.0, 0], "kkt": [0.0, 0], "prec": [0.0, 0]}
    flush.fill_(1.0)
    torch.cuda.synchronize()
    for i in range(len(cs)):
        ctxs[i].profile(True)
        oc.ipm_solve(probs[i], params, outputs=outs[i])
        pr = ctxs[i].profile_read()
        ctxs[i].profile(False)
        for k in prof:
            prof[k][0] += pr[k][0]
            prof[k][1] += pr[k][1]
    peak, peak_src = measured_peak_hbm()
    sweep_ms, sweep_n = prof["sweep"]
    fuse = C.c_int(0)
    _lib.check(_lib.load().oc_get_tuning(b"sweep_fuse", C.byref(fuse)))
    fuse = max(1, min(5, fuse.value))
    # the sampled launch fuses `fuse` sweeps; the byte model counts 4V per sweep
    sweep_bytes = fuse * bytes_model.sweep_bytes(ny)
    traffic = measured_traffic(args.level, fuse)
    achieved = sweep_bytes / (sweep_ms / sweep_n / 1e3) / 1e9 if sweep_n else None
    kkt_b, prec_b = bytes_model.apply_bytes("pt" if args.solver == "gmres-pt" else "pd",
                                            args.level, ny)
    # KKT + preconditioner apply as the solver runs it (preconditioner graph
    # replayed, 20 applies on cell 0's last Newton state, CUDA events on its
    # stream); the per-launch event pass above disables graph capture
    kind = "pt" if args.solver == "gmres-pt" else "pd"
    kkt_ms, prec_ms = probs[0].time_applies(kind, 20)
    kkt_n = prec_n = 1
    apply_gbs = (kkt_b + prec_b) / ((kkt_ms + prec_ms) / 1e3) / 1e9

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            v, cores, kind, sample, _, _ = cpu_reference_sample(args.level, args.solver)
            cpu = {"value": v, "unit": UNIT, "cores": cores, "kind": kind, "sample": sample}
        except Exception as e:
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "port",
                   "sample": f"unavailable: {e}"}

    if rank == 0:
        ipm_ms = [r.solve_ms for r in results]
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": max_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded sine-mode y_d; no dataset exists for this path)",
            "config": workload(args.level, args.solver),
            "roofline": {
                "bound": "hbm",
                "kernel": f"k_sweep (fine-level 4-colour GS, {fuse} fused sweeps per launch)",
                "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": (achieved / peak) if achieved else None,
                "traffic": traffic["bytes"] if traffic else None,
                "traffic_source": traffic["source"] if traffic else None,
                "peak_source": peak_src,
                "bytes_per_launch": sweep_bytes,
                "avg_launch_ms": sweep_ms / sweep_n if sweep_n else None,
                "launches_in_pass": sweep_n,
                "note": "per-launch CUDA events on the solver stream, cells run one at a time; "
                        "level-9 fields (2 MiB) are L2-resident between sweeps; traffic = DRAM "
                        "read+write of the same launch from ncu (cold cache), see profiles/",
            },
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h),
                    "what": "build_qp from pinned host arrays (upload, device setup), "
                            "ipm_solve, u/y/z/p to pinned host arrays, close; 9 cells per "
                            "step, concurrent"},
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
            "ipm_time_to_tolerance_ms": {"mean": statistics.mean(ipm_ms), "max": max(ipm_ms),
                                         "note": "per cell, 9 cells in flight"},
            "nli": [r.stats.nli for r in results],
            "av_li": [round(r.stats.av_li, 3) for r in results],
            "ipm_solves_per_s": len(results) * world * 1e3 * args.steps / max_ms,
            "iteration_note": "the default 4-colour smoother needs more Krylov iterations per "
                              "Newton step than the reference's lexicographic GS on this "
                              "workload (av_li 4.67 vs 4.22, profiles/r01/parity_full.json): "
                              "time-to-solution gains are the it/s ratio x 4.22/4.67",
            "kkt_precond_apply": {"gbs": apply_gbs, "kkt_ms": kkt_ms / kkt_n if kkt_n else None,
                                  "prec_ms": prec_ms / prec_n if prec_n else None,
                                  "bytes": kkt_b + prec_b, "frac_of_peak":
                                  (apply_gbs / peak) if apply_gbs else None,
                                  "how": "oc_time_applies on cell 0's last Newton state: 20 graph-"
                                         "replayed applies, other cells idle but their contexts "
                                         "live (launch shapes for 9 concurrent cells; alone: "
                                         "tools/apply_bw.py); SURVEY 8d byte model"},
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
