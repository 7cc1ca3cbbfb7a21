"""Benchmark harness on the device backend: the reference's
`run_benchmark` / `run_sweep` callers of the hot path and their CSV artefacts
(bench.hpp:17-90, bench.cpp:150-382), driving `optcon.ipm_solve` instead of the
CPU solver. Same configuration fields and defaults, same file names, columns and
number formatting (`%.17g`), same sweep presets; reruns are bit-identical
(the device reductions use a fixed order).

    from paper_1806_05896_b200 import harness
    art = harness.run_benchmark(harness.RunConfig(pde="poisson", ell=6, out_dir="out"))
    harness.run_sweep(harness.sweep_preset("table1"), "table1.csv")
"""
from __future__ import annotations

import math
import os
import threading
import time
from dataclasses import dataclass, field, replace
from typing import List, Optional, Tuple

import numpy as np

from . import optcon as oc

PDES = ("poisson", "convdiff", "heat")
SOLVERS = ("gmres-pt", "minres-pd", "gmres-ppi")


@dataclass
class RunConfig:
    """bench.hpp:17-37 (defaults included)."""

    pde: str = "poisson"
    ell: int = 5
    alpha: float = 1e-2
    beta: float = 1e-2
    sigma: float = 0.2
    eps: float = 1e-1
    tau: float = 0.04
    horizon: float = 1.0
    solver: str = "gmres-pt"
    ua: float = -2.0
    ub: float = 1.5
    ya: Optional[float] = None
    yb: Optional[float] = None
    obs_box: Optional[Tuple[float, float, float, float]] = None
    lintol: float = 1e-10
    mu0: float = 1.0
    max_iterations: int = 100
    out_dir: str = "."
    dump_solution: bool = False
    label: str = ""
    smoother: str = "color4"  # device option: "lex" reproduces the reference's Krylov counts


@dataclass
class RunArtifacts:
    """bench.hpp:39-50."""

    stats: oc.IpmStats
    sparsity: oc.SparsityReport
    converged: bool
    stats_csv: str
    summary_csv: str
    solution_csv: str = ""
    wall_seconds: float = 0.0


@dataclass
class SweepSpec:
    """bench.hpp:68-75."""

    base: RunConfig = field(default_factory=RunConfig)
    ells: List[int] = field(default_factory=list)
    alphas: List[float] = field(default_factory=list)
    betas: List[float] = field(default_factory=list)
    epss: List[float] = field(default_factory=list)
    taus: List[float] = field(default_factory=list)


def fmt(v: float) -> str:
    """bench.cpp:19-24: printf("%.17g")."""
    return "%.17g" % v


def config_from_map(kv: dict) -> RunConfig:
    """bench.cpp config_from_map: key=value strings to a RunConfig."""
    c = RunConfig()
    conv = dict(ell=int, alpha=float, beta=float, sigma=float, eps=float, tau=float,
                ua=float, ub=float, ya=float, yb=float, lintol=float, mu0=float)
    for k, v in kv.items():
        if k == "pde":
            if v not in PDES:
                raise oc.OptconInvalidArgument("unknown pde: " + v)
            c.pde = v
        elif k == "solver":
            if v not in SOLVERS:
                raise oc.OptconInvalidArgument("unknown solver: " + v)
            c.solver = v
        elif k == "T":
            c.horizon = float(v)
        elif k == "out":
            c.out_dir = v
        elif k == "obs_box":
            parts = v.split(",")
            if len(parts) < 4:
                raise oc.OptconInvalidArgument("obs_box needs 4 values")
            c.obs_box = tuple(float(p) for p in parts[:4])
        elif k in conv:
            setattr(c, k, conv[k](v))
    return c


def validate_config(cfg: RunConfig) -> None:
    """bench.cpp validate_config (messages verbatim)."""
    if cfg.obs_box is not None and cfg.solver != "gmres-ppi":
        raise oc.OptconInvalidArgument(
            "partial observation makes the (1,1)-block singular: use --solver gmres-ppi")
    if cfg.obs_box is None and cfg.solver == "gmres-ppi" and cfg.pde == "heat":
        raise oc.OptconInvalidArgument("gmres-ppi is not available for heat problems")
    if cfg.pde == "heat" and cfg.solver != "gmres-pt":
        raise oc.OptconInvalidArgument("heat problems support --solver gmres-pt only")
    if (cfg.ya is None) != (cfg.yb is None):
        raise oc.OptconInvalidArgument("state bounds must be given as a pair (--ya and --yb)")
    if cfg.ell < 3 or cfg.ell > 12:
        raise oc.OptconInvalidArgument("ell out of supported range")


def default_desired_state(pde: str, ell: int) -> np.ndarray:
    """bench.cpp default_desired_state interpolated at the interior nodes:
    a Gaussian bump for convection-diffusion, sin(pi x) sin(pi y) otherwise."""
    nx = (1 << ell) - 1
    h = 1.0 / (1 << ell)
    out = np.empty(nx * nx)
    for gy in range(nx):
        y = (gy + 1) * h
        for gx in range(nx):
            x = (gx + 1) * h
            if pde == "convdiff":
                out[gy * nx + gx] = math.exp(-64.0 * ((x - 0.5) * (x - 0.5) + (y - 0.5) * (y - 0.5)))
            else:
                out[gy * nx + gx] = math.sin(math.pi * x) * math.sin(math.pi * y)
    return out


def nodal_sparsity(u_interior, ell: int, nt: int = 1, threshold: float = 1e-2):
    """bench.cpp nodal_sparsity: percentage of |u| < threshold over the full
    nodal function (boundary nodes carry zero control) and the l1 norm of u."""
    nx = (1 << ell) - 1
    full = (nx + 2) * (nx + 2)
    u = np.asarray(u_interior, dtype=np.float64)
    if u.size != nx * nx * nt:
        raise oc.OptconInvalidArgument("nodal_sparsity: size does not match level")
    below = int(np.count_nonzero(np.abs(u) < threshold)) + (full - nx * nx) * nt
    l1 = 0.0
    for v in u:  # sequential sum, as the reference loop
        l1 += abs(float(v))
    return oc.SparsityReport(100.0 * below / float(full * nt), l1)


def summary_header() -> str:
    return "pde,ell,alpha,beta,sigma,eps,tau,solver,nli,av_li,sparsity,l1,converged"


def summary_row(cfg: RunConfig, stats: oc.IpmStats, sp: oc.SparsityReport, converged: bool) -> str:
    return ",".join([cfg.pde, str(cfg.ell), fmt(cfg.alpha), fmt(cfg.beta), fmt(cfg.sigma),
                     fmt(cfg.eps), fmt(cfg.tau if cfg.pde == "heat" else 0.0), cfg.solver,
                     str(stats.nli), fmt(stats.av_li), fmt(sp.percent_below_threshold),
                     fmt(sp.l1_norm), "1" if converged else "0"])


def write_stats_csv(path: str, stats: oc.IpmStats, heat: bool, tau: float) -> None:
    with open(path, "w") as f:
        f.write("k,mu,xi_p,xi_d,xi_c,lin_iters,lin_relres" + (",tau\n" if heat else "\n"))
        for it in stats.iterations:
            row = ",".join([str(it.k), fmt(it.mu), fmt(it.norm_xp), fmt(it.norm_xd),
                            fmt(it.norm_xc), str(it.lin_iters), fmt(it.lin_relres)])
            f.write(row + ("," + fmt(tau) if heat else "") + "\n")


def dump_solution_csv(path: str, ell: int, u, state) -> None:
    """Full nodal field, boundary nodes carrying the Dirichlet zeros."""
    nx = (1 << ell) - 1
    h = 1.0 / (1 << ell)
    with open(path, "w") as f:
        f.write("x,y,u,state\n")
        for gy in range(nx + 2):
            for gx in range(nx + 2):
                uv = yv = 0.0
                if 1 <= gx <= nx and 1 <= gy <= nx:
                    i = (gy - 1) * nx + (gx - 1)
                    uv, yv = float(u[i]), float(state[i])
                f.write(f"{fmt(gx * h)},{fmt(gy * h)},{fmt(uv)},{fmt(yv)}\n")


def _problem(cfg: RunConfig) -> oc.ControlProblem:
    kw = dict(pde=cfg.pde, alpha=cfg.alpha, beta=cfg.beta, y_d=default_desired_state(cfg.pde, cfg.ell),
              u_a=cfg.ua, u_b=cfg.ub)
    if cfg.pde == "convdiff":
        kw["eps"] = cfg.eps
    if cfg.pde == "heat":
        kw.update(tau=cfg.tau, horizon=cfg.horizon)
    if cfg.ya is not None:
        kw.update(y_a=cfg.ya, y_b=cfg.yb)
    if cfg.obs_box is not None:
        kw["observation"] = tuple(cfg.obs_box)
    return oc.ControlProblem(**kw)


def _params(cfg: RunConfig) -> oc.IpmParams:
    return oc.IpmParams(sigma=cfg.sigma, solver=cfg.solver, linear_tol=cfg.lintol, mu0=cfg.mu0,
                        max_iterations=cfg.max_iterations, smoother=cfg.smoother)


def _solve(cfg: RunConfig, ctx: oc.Context):
    problem = _problem(cfg)
    grid = oc.Grid(cfg.ell)
    qp = (oc.assemble_spacetime if cfg.pde == "heat" else oc.build_qp)(problem, grid, ctx)
    try:
        r = oc.ipm_solve(qp, _params(cfg))
        nt = qp.nt
    finally:
        qp.close()
    return r, nt


def run_benchmark(cfg: RunConfig, ctx: Optional[oc.Context] = None) -> RunArtifacts:
    """bench.cpp run_benchmark: one solve, stats.csv + summary.csv (+ solution.csv)."""
    validate_config(cfg)
    t0 = time.perf_counter()
    os.makedirs(cfg.out_dir, exist_ok=True)
    r, nt = _solve(cfg, ctx or oc.default_context())
    sp = nodal_sparsity(r.u, cfg.ell, nt)
    art = RunArtifacts(stats=r.stats, sparsity=sp, converged=r.stats.converged,
                       stats_csv=os.path.join(cfg.out_dir, "stats.csv"),
                       summary_csv=os.path.join(cfg.out_dir, "summary.csv"))
    if cfg.dump_solution:
        nn = ((1 << cfg.ell) - 1) ** 2
        off = nn * (nt - 1)  # heat: terminal time slice
        art.solution_csv = os.path.join(cfg.out_dir, "solution.csv")
        dump_solution_csv(art.solution_csv, cfg.ell, r.u[off:off + nn], r.state.y[off:off + nn])
    write_stats_csv(art.stats_csv, r.stats, cfg.pde == "heat", cfg.tau)
    with open(art.summary_csv, "w") as f:
        f.write(summary_header() + "\n" + summary_row(cfg, r.stats, sp, art.converged) + "\n")
    art.wall_seconds = time.perf_counter() - t0
    return art


def sweep_cells(spec: SweepSpec) -> List[RunConfig]:
    cells = []
    for ell in spec.ells:
        for alpha in spec.alphas:
            if spec.betas:
                vary = [replace(spec.base, beta=b) for b in spec.betas]
            elif spec.epss:
                vary = [replace(spec.base, eps=e) for e in spec.epss]
            elif spec.taus:
                vary = [replace(spec.base, tau=t) for t in spec.taus]
            else:
                vary = [replace(spec.base)]
            cells += [replace(c, ell=ell, alpha=alpha) for c in vary]
    return cells


def run_sweep(spec: SweepSpec, csv_path: str, workers: Optional[int] = None) -> int:
    """bench.cpp run_sweep: every cell solved (cells run concurrently, one
    device context per worker thread, like the reference's thread pool), one
    summary row per cell in cell order."""
    cells = sweep_cells(spec)
    rows = [""] * len(cells)
    nworkers = min(workers or int(os.environ.get("SOLVER_THREADS", "9")), max(len(cells), 1))
    nxt = [0]
    lock = threading.Lock()
    errors = []

    def worker():
        ctx = oc.Context(0)
        while True:
            with lock:
                i = nxt[0]
                nxt[0] += 1
            if i >= len(cells):
                return
            try:
                cfg = cells[i]
                validate_config(cfg)
                r, nt = _solve(cfg, ctx)
                rows[i] = summary_row(cfg, r.stats, nodal_sparsity(r.u, cfg.ell, nt),
                                      r.stats.converged)
            except Exception as e:  # surfaced after the pool drains
                errors.append(e)
                return

    pool = [threading.Thread(target=worker) for _ in range(nworkers)]
    for t in pool:
        t.start()
    for t in pool:
        t.join()
    if errors:
        raise errors[0]
    with open(csv_path, "w") as f:
        f.write(summary_header() + "\n")
        for r in rows:
            f.write(r + "\n")
    return len(cells)


def sweep_preset(name: str) -> SweepSpec:
    """bench.cpp sweep_preset: the paper's tables."""
    if name == "table1":
        return SweepSpec(RunConfig(pde="poisson", sigma=0.2), [5], [1e-2, 1e-4, 1e-6],
                         betas=[1e-1, 1e-2, 1e-3])
    if name == "table2":
        return SweepSpec(RunConfig(pde="poisson", sigma=0.2, beta=1e-2), [6, 7, 8, 9],
                         [1e-2, 1e-4, 1e-6])
    if name == "table3":
        return SweepSpec(RunConfig(pde="convdiff", beta=1e-3, sigma=0.25), [6, 7, 8, 9],
                         [1e-2, 1e-4, 1e-6], epss=[1e-1])
    if name == "table3b":
        return SweepSpec(RunConfig(pde="convdiff", beta=1e-3, sigma=0.4), [6, 7, 8, 9],
                         [1e-2, 1e-4, 1e-6], epss=[1e-2])
    if name == "table4":
        return SweepSpec(RunConfig(pde="poisson", sigma=0.2, beta=1e-2, ua=-1.0, ub=15.0,
                                   ya=-0.1, yb=0.8), [6, 7, 8, 9], [1e-2, 1e-4, 1e-6])
    if name == "table6":
        return SweepSpec(RunConfig(pde="heat", sigma=0.25, beta=1e-2), [4, 5, 6],
                         [1e-2, 1e-4, 1e-6], taus=[0.04, 0.02, 0.01])
    raise oc.OptconInvalidArgument("unknown sweep preset: " + name)
