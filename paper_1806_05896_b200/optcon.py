"""Python mirror of the reference optcon solver API over the B200 C-ABI.

Names, argument meaning and error behaviour follow the reference C++ headers
(/root/reference/proj/include/optcon): ``ControlProblem`` (qp.hpp:20-34),
``build_qp`` (qp.hpp:82), ``assemble_spacetime`` (timedep.hpp:68),
``IpmParams`` (ipm.hpp:17-32), ``ipm_solve`` (ipm.hpp:134), ``IpmResult``
(ipm.hpp:100-105), ``make_saddle_operator`` (ipm.hpp:138),
``MgHierarchy`` (multigrid.hpp:43-64), ``ChebyshevSemiIteration``
(chebyshev.hpp:17-37). ``std::invalid_argument`` surfaces as
``OptconInvalidArgument`` (a ValueError), ``std::runtime_error`` as
``OptconError``. All compute happens in sm_100a kernels through
``_lib/liboptcon_b200.so``; arrays may be numpy (host) or torch CUDA tensors
(device, used in place without copies).
"""
from __future__ import annotations

import atexit
import ctypes as C
import weakref
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _lib
from ._lib import OptconCudaError, OptconError, OptconInvalidArgument  # noqa: F401

PDES = {"poisson": 0, "convdiff": 1, "heat": 2}
SOLVERS = {"gmres-pt": 0, "minres-pd": 1, "gmres-ppi": 2}
PRECONDS = {"pd": 0, "pt": 1, "ppi": 2}


def _is_torch(a) -> bool:
    return type(a).__module__.startswith("torch")


class _Arg:
    """Keeps host arrays alive while their pointer is in use."""

    def __init__(self):
        self.keep = []

    def ptr(self, a, size: Optional[int] = None):
        if a is None:
            return None
        if _is_torch(a):
            import torch

            if a.dtype != torch.float64 or not a.is_contiguous():
                raise OptconInvalidArgument("tensor arguments must be contiguous float64")
            if size is not None and a.numel() != size:
                raise OptconInvalidArgument(f"expected {size} entries, got {a.numel()}")
            return C.c_void_p(a.data_ptr())
        arr = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
        if size is not None:
            if arr.size == 1 and size != 1:
                arr = np.full(size, float(arr.reshape(-1)[0]))
            if arr.size != size:
                raise OptconInvalidArgument(f"expected {size} entries, got {arr.size}")
        self.keep.append(arr)
        return C.c_void_p(arr.ctypes.data)


# Device objects still alive at interpreter exit are closed before module
# teardown (problems and hierarchies before their contexts): left to the
# finaliser, a context could otherwise be destroyed after the CUDA runtime.
_live_objects: "weakref.WeakSet" = weakref.WeakSet()
_live_contexts: "weakref.WeakSet" = weakref.WeakSet()


@atexit.register
def _close_live_objects():
    for o in list(_live_objects):
        try:
            o.close()
        except Exception:
            pass
    for c in list(_live_contexts):
        try:
            c.close()
        except Exception:
            pass


class Context:
    """One device context (CUDA stream + pinned scalars) per host thread."""

    def __init__(self, device: int = 0):
        self._L = _lib.load()
        h = C.c_void_p()
        _lib.check(self._L.oc_create(C.byref(h), device))
        self.h = h
        self.device = device
        _live_contexts.add(self)

    def synchronize(self):
        _lib.check(self._L.oc_synchronize(self.h))

    # instrumentation (bench)
    def record(self, slot: int):
        """Record CUDA event `slot` (0..7) on the solver stream."""
        _lib.check(self._L.oc_event_record(self.h, slot))

    def elapsed_ms(self, a: int, b: int) -> float:
        ms = C.c_double()
        _lib.check(self._L.oc_event_elapsed(self.h, a, b, C.byref(ms)))
        return ms.value

    def elapsed_ms_to(self, a: int, other: "Context", b: int) -> float:
        """ms from this context's event `a` to `other`'s event `b` (same device)."""
        ms = C.c_double()
        _lib.check(self._L.oc_event_elapsed_between(self.h, a, other.h, b, C.byref(ms)))
        return ms.value

    def profile(self, enable: bool):
        _lib.check(self._L.oc_profile(self.h, int(enable)))

    def profile_read(self):
        """{"sweep"|"kkt"|"prec"|"block": (total_ms, count)} since the last read."""
        ms = (C.c_double * 4)()
        cnt = (C.c_longlong * 4)()
        _lib.check(self._L.oc_profile_read(self.h, ms, cnt))
        return {k: (ms[i], cnt[i]) for i, k in enumerate(("sweep", "kkt", "prec", "block"))}

    @staticmethod
    def launch_count() -> int:
        return int(_lib.load().oc_launch_count())

    def close(self):
        if getattr(self, "h", None):
            self._L.oc_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default_ctx: Optional[Context] = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


class Grid:
    """grid.hpp:14-37: h = 2^-level, (2^level - 1)^2 interior nodes, x fastest."""

    def __init__(self, level: int):
        if level < 1 or level > 14:
            raise OptconInvalidArgument("Grid: level out of range")
        self.level = level

    @property
    def h(self) -> float:
        return 1.0 / (1 << self.level)

    def nx(self) -> int:
        return (1 << self.level) - 1

    def num_nodes(self) -> int:
        return self.nx() ** 2

    def node_xy(self):
        nx = self.nx()
        idx = np.arange(nx * nx)
        return (idx % nx + 1) * self.h, (idx // nx + 1) * self.h


@dataclass
class ControlProblem:
    """qp.hpp:20-34 (nodal data at interior nodes)."""

    pde: str = "poisson"
    eps: float = 1e-1
    tau: float = 0.04
    horizon: float = 1.0
    alpha: float = 1e-2
    beta: float = 1e-2
    y_d: object = None
    f: object = None
    u_a: object = None
    u_b: object = None
    y_a: object = None
    y_b: object = None
    observation: Optional[Sequence[float]] = None  # (a1, b1, a2, b2)


SMOOTHERS = {"color4": 0, "lex": 1, "auto": 2}


def smoother_id(s) -> int:
    """'auto' (default: colour sweeps, lexicographic after a capped solve), 'color4'
    (4-colour symmetric GS) or 'lex' (the reference's
    lexicographic GS, multigrid.cpp:44-66, faithful mode); ints pass through."""
    if isinstance(s, str):
        if s not in SMOOTHERS:
            raise OptconInvalidArgument(f"unknown smoother: {s}")
        return SMOOTHERS[s]
    return int(s)


@dataclass
class IpmParams:
    """ipm.hpp:17-32 (+ gmres_restart, smoother)."""

    alpha0: float = 0.995
    sigma: float = 0.2
    eps_p: float = 1e-6
    eps_d: float = 1e-6
    eps_c: float = 1e-6
    mu0: float = 1.0
    max_iterations: int = 100
    linear_tol: float = 1e-10
    linear_maxit: int = 200
    cheb_steps: int = 20
    mg_cycles: int = 3
    mg_pre: int = 5
    mg_post: int = 5
    solver: str = "gmres-pt"
    # "auto" (default): colour sweeps, lexicographic from the first Newton solve
    # capped at linear_maxit on (that solve redone); "color4"; "lex" (faithful)
    smoother: object = "auto"
    gmres_restart: int = 0

    def c(self) -> _lib.IpmParamsC:
        if self.solver not in SOLVERS:
            raise OptconInvalidArgument(f"unknown solver: {self.solver}")
        return _lib.IpmParamsC(
            self.alpha0, self.sigma, self.eps_p, self.eps_d, self.eps_c, self.mu0,
            int(self.max_iterations), self.linear_tol, int(self.linear_maxit),
            int(self.cheb_steps), int(self.mg_cycles), int(self.mg_pre), int(self.mg_post),
            SOLVERS[self.solver], smoother_id(self.smoother), int(self.gmres_restart))


@dataclass
class IterationRecord:
    k: int
    mu: float
    norm_xp: float
    norm_xd: float
    norm_xc: float
    lin_iters: int
    lin_relres: float
    lin_converged: bool
    newton_ms: float = 0.0


@dataclass
class IpmStats:
    iterations: list = field(default_factory=list)
    converged: bool = False
    nli: int = 0
    av_li: float = 0.0


@dataclass
class SparsityReport:
    percent_below_threshold: float
    l1_norm: float


@dataclass
class IpmState:
    y: np.ndarray
    z: np.ndarray
    p: np.ndarray
    lam_ya: Optional[np.ndarray]
    lam_yb: Optional[np.ndarray]
    lam_za: np.ndarray
    lam_zb: np.ndarray
    mu: float
    k: int


@dataclass
class IpmResult:
    state: IpmState
    u: np.ndarray
    sparsity: SparsityReport
    stats: IpmStats
    objective: float
    nodal_sparsity: float
    total_lin: int
    solve_ms: float
    newton_ms: float
    discarded_lin: int = 0  # auto smoother: iterations of capped colour solves redone
    lex_from: int = 0       # first Newton step solved with the lexicographic smoother


@dataclass
class SolveReport:
    iterations: int
    relative_residual: float
    converged: bool
    breakdown: bool
    message: str


@dataclass
class ThetaBlocks:
    """precond.hpp:16-20; theta_y may be None (no state box)."""

    theta_y: Optional[np.ndarray]
    theta_w: np.ndarray
    theta_v: np.ndarray


class QpProblem:
    """Device-resident problem (QpProblem / SpaceTimeSystem) with its solver."""

    def __init__(self, problem: ControlProblem, grid: Grid, ctx: Optional[Context] = None):
        self.ctx = ctx or default_context()
        self._L = self.ctx._L
        if problem.pde not in PDES:
            raise OptconInvalidArgument(f"unknown pde: {problem.pde}")
        n = grid.num_nodes()
        a = _Arg()
        d = _lib.ProblemDesc()
        d.pde = PDES[problem.pde]
        d.level = grid.level
        d.eps = problem.eps
        d.tau = problem.tau
        d.horizon = problem.horizon
        d.quadrature = 0
        d.alpha = problem.alpha
        d.beta = problem.beta
        yd = problem.y_d
        yd_len = int(yd.numel() if _is_torch(yd) else np.asarray(yd).size)
        d.y_d = a.ptr(yd)
        d.y_d_len = yd_len
        d.f = a.ptr(problem.f, n)
        d.u_a = a.ptr(problem.u_a, n)
        d.u_b = a.ptr(problem.u_b, n)
        if (problem.y_a is None) != (problem.y_b is None):
            raise OptconInvalidArgument("ControlProblem: state bounds must come as a pair")
        d.y_a = a.ptr(problem.y_a, n)
        d.y_b = a.ptr(problem.y_b, n)
        if problem.observation is not None:
            d.has_obs = 1
            for i in range(4):
                d.obs[i] = float(problem.observation[i])
        h = C.c_void_p()
        _lib.check(self._L.oc_problem_create(self.ctx.h, C.byref(d), C.byref(h)))
        self.h = h
        _live_objects.add(self)
        info = _lib.ProblemInfoC()
        _lib.check(self._L.oc_problem_info_get(self.h, C.byref(info)))
        self.n, self.nt, self.ny = info.n, info.nt, info.ny
        self.has_state_bounds = bool(info.has_state_bounds)
        self.partial_observation = bool(info.partial_observation)
        self.level = info.level
        self.h2d_bytes = int(info.h2d_bytes)
        self.grid = grid
        self.problem = problem

    def close(self):
        if getattr(self, "h", None):
            self._L.oc_problem_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------ components
    def kkt_apply(self, theta: ThetaBlocks, x):
        """make_saddle_operator(model, theta).apply(x) (ipm.cpp:237-268)."""
        a = _Arg()
        out = np.zeros(4 * self.ny)
        _lib.check(self._L.oc_kkt_apply(
            self.h, a.ptr(theta.theta_y, self.ny) if theta.theta_y is not None else None,
            a.ptr(theta.theta_w, self.ny), a.ptr(theta.theta_v, self.ny), a.ptr(x, 4 * self.ny),
            a.ptr(out)))
        return a.keep[-1]

    def precond_setup(self, theta: ThetaBlocks, params: IpmParams):
        a = _Arg()
        pc = params.c()
        _lib.check(self._L.oc_precond_setup(
            self.h, a.ptr(theta.theta_y, self.ny) if theta.theta_y is not None else None,
            a.ptr(theta.theta_w, self.ny), a.ptr(theta.theta_v, self.ny), C.byref(pc)))

    def precond_apply(self, kind: str, r):
        a = _Arg()
        rp = a.ptr(r, 4 * self.ny)
        out = np.zeros(4 * self.ny)
        op = a.ptr(out)
        _lib.check(self._L.oc_precond_apply(self.h, PRECONDS[kind], rp, op))
        return a.keep[-1]

    def schur_apply(self, r):
        a = _Arg()
        rp = a.ptr(r, self.ny)
        out = np.zeros(self.ny)
        op = a.ptr(out)
        _lib.check(self._L.oc_schur_apply(self.h, rp, op))
        return a.keep[-1]

    def newton_solve(self, theta: ThetaBlocks, r1, r2, r3, params: IpmParams):
        """IpmModel::newton_solve (ipm.cpp:394-468)."""
        a = _Arg()
        pc = params.c()
        dy, dz, dp = np.zeros(self.ny), np.zeros(2 * self.ny), np.zeros(self.ny)
        rep = _lib.SolveReportC()
        _lib.check(self._L.oc_newton_solve(
            self.h, a.ptr(theta.theta_y, self.ny) if theta.theta_y is not None else None,
            a.ptr(theta.theta_w, self.ny), a.ptr(theta.theta_v, self.ny), a.ptr(r1, self.ny),
            a.ptr(r2, 2 * self.ny), a.ptr(r3, self.ny), C.byref(pc), a.ptr(dy), a.ptr(dz),
            a.ptr(dp), C.byref(rep)))
        return dy, dz, dp, SolveReport(rep.iterations, rep.relative_residual,
                                       bool(rep.converged), bool(rep.breakdown),
                                       rep.message.decode())

    def ipm_pieces(self, y, z, p, lam_za, lam_zb, lam_ya=None, lam_yb=None, mu_state=1.0,
                   mu_rhs=0.2):
        """build_theta + newton_rhs + ipm_residuals (ipm.cpp:32-143)."""
        a = _Arg()
        ny = self.ny
        outs = [np.zeros(ny), np.zeros(ny), np.zeros(ny), np.zeros(ny), np.zeros(2 * ny),
                np.zeros(ny), np.zeros(3)]
        ptrs = [a.ptr(o) for o in outs]
        _lib.check(self._L.oc_ipm_pieces(
            self.h, a.ptr(y, ny), a.ptr(z, 2 * ny), a.ptr(p, ny),
            a.ptr(lam_ya, ny) if lam_ya is not None else None,
            a.ptr(lam_yb, ny) if lam_yb is not None else None, a.ptr(lam_za, 2 * ny),
            a.ptr(lam_zb, 2 * ny), C.c_double(mu_state), C.c_double(mu_rhs), *ptrs))
        return dict(theta_y=outs[0], theta_w=outs[1], theta_v=outs[2], r1=outs[3], r2=outs[4],
                    r3=outs[5], norms=outs[6])

    def objective(self, y, z) -> float:
        a = _Arg()
        o = C.c_double()
        _lib.check(self._L.oc_objective(self.h, a.ptr(y, self.ny), a.ptr(z, 2 * self.ny),
                                        C.byref(o)))
        return o.value

    def time_applies(self, kind: str, reps: int = 20):
        """Device ms of one KKT apply and one preconditioner apply (CUDA events)."""
        k, p = C.c_double(), C.c_double()
        _lib.check(self._L.oc_time_applies(self.h, PRECONDS[kind], reps, C.byref(k), C.byref(p)))
        return k.value, p.value


def build_qp(problem: ControlProblem, grid: Grid, ctx: Optional[Context] = None) -> QpProblem:
    """qp.hpp:82 — assemble and upload the QP; rejects the heat PDE."""
    if problem.pde == "heat":
        raise OptconInvalidArgument("build_qp: heat problems use the space-time assembly")
    return QpProblem(problem, grid, ctx)


def assemble_spacetime(problem: ControlProblem, grid: Grid,
                       ctx: Optional[Context] = None) -> QpProblem:
    """timedep.hpp:68 — backward-Euler space-time system (heat only)."""
    if problem.pde != "heat":
        raise OptconInvalidArgument("assemble_spacetime: expects the heat problem")
    return QpProblem(problem, grid, ctx)


def ipm_solve(qp: QpProblem, params: IpmParams = IpmParams(), outputs=None) -> IpmResult:
    """ipm.hpp:134 — the whole interior-point loop on the device.

    ``outputs`` may supply preallocated arrays (numpy or torch CUDA tensors) for
    any of y, z, p, u, lam_za, lam_zb, lam_ya, lam_yb."""
    L = qp._L
    ny = qp.ny
    a = _Arg()
    o = dict(outputs or {})
    names = ["y", "z", "p", "lam_ya", "lam_yb", "lam_za", "lam_zb", "u"]
    sizes = dict(y=ny, z=2 * ny, p=ny, lam_ya=ny, lam_yb=ny, lam_za=2 * ny, lam_zb=2 * ny, u=ny)
    for k in names:
        if k not in o:
            if k in ("lam_ya", "lam_yb") and not qp.has_state_bounds:
                o[k] = None
            else:
                o[k] = np.zeros(sizes[k])
    ptrs = {}
    for k in names:
        if o[k] is None:
            ptrs[k] = None
        elif _is_torch(o[k]):
            ptrs[k] = a.ptr(o[k], sizes[k])
        else:
            arr = o[k]
            assert arr.dtype == np.float64 and arr.flags.c_contiguous and arr.size == sizes[k]
            ptrs[k] = C.c_void_p(arr.ctypes.data)
    cap = max(params.max_iterations + 1, 1)
    recs = (_lib.IterRecordC * cap)()
    r = _lib.IpmResultC()
    for k in names:
        setattr(r, k, ptrs[k])
    r.records = C.cast(recs, C.POINTER(_lib.IterRecordC))
    r.records_cap = cap
    pc = params.c()
    _lib.check(L.oc_ipm_solve(qp.h, C.byref(pc), C.byref(r)))
    its = [IterationRecord(recs[i].k, recs[i].mu, recs[i].norm_xp, recs[i].norm_xd,
                           recs[i].norm_xc, recs[i].lin_iters, recs[i].lin_relres,
                           bool(recs[i].lin_converged), recs[i].newton_ms)
           for i in range(min(r.n_records, cap))]
    stats = IpmStats(its, bool(r.converged), r.nli, r.av_li)
    state = IpmState(o["y"], o["z"], o["p"], o["lam_ya"], o["lam_yb"], o["lam_za"],
                     o["lam_zb"], r.mu, r.nli)
    return IpmResult(state, o["u"], SparsityReport(r.sparsity_pct, r.l1), stats, r.objective,
                     r.nodal_sparsity_pct, r.total_lin, r.solve_ms, r.newton_ms,
                     r.discarded_lin, r.lex_from)


def solve_heat_control(problem: ControlProblem, grid: Grid, params: IpmParams = IpmParams(),
                       ctx: Optional[Context] = None) -> IpmResult:
    """timedep.hpp:88-91."""
    return ipm_solve(assemble_spacetime(problem, grid, ctx), params)


def recover_control(z):
    """qp.hpp:40 — u = w - v (host helper on results)."""
    z = np.asarray(z)
    if z.size % 2:
        raise OptconInvalidArgument("recover_control: odd length")
    n = z.size // 2
    return z[:n] - z[n:]


class MgHierarchy:
    """multigrid.hpp:43-64 over an explicit 9-point operator (9 x n arrays)."""

    def __init__(self, coef9, level: int, rediscretize: int = 0, eps: float = 0.1,
                 ctx: Optional[Context] = None, smoother="color4"):
        self.ctx = ctx or default_context()
        self._L = self.ctx._L
        self.level = level
        self.n = ((1 << level) - 1) ** 2
        a = _Arg()
        h = C.c_void_p()
        _lib.check(self._L.oc_mg_create(self.ctx.h, level, a.ptr(np.ravel(coef9), 9 * self.n),
                                        rediscretize, C.c_double(eps), smoother_id(smoother),
                                        C.byref(h)))
        self.h = h
        _live_objects.add(self)

    def close(self):
        if getattr(self, "h", None):
            self._L.oc_mg_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def solve(self, rhs, cycles=3, pre=5, post=5):
        a = _Arg()
        rp = a.ptr(rhs, self.n)
        out = np.zeros(self.n)
        _lib.check(self._L.oc_mg_solve(self.h, rp, cycles, pre, post, a.ptr(out)))
        return a.keep[-1]

    def depth(self) -> int:
        return self._L.oc_mg_depth(self.h)

    def level_matrix(self, k: int):
        nx = (1 << (self.level - k)) - 1
        out = np.zeros(9 * nx * nx)
        _lib.check(self._L.oc_mg_level_matrix(self.h, k, C.c_void_p(out.ctypes.data)))
        return out.reshape(9, nx * nx)

    def smooth(self, b, x, forward=True):
        a = _Arg()
        bp = a.ptr(b, self.n)
        xx = np.array(x, dtype=np.float64, copy=True)
        _lib.check(self._L.oc_mg_smooth(self.h, bp, C.c_void_p(xx.ctypes.data), int(forward)))
        return xx


def cheb_apply(level: int, scale: float, extra, steps: int, b, ctx: Optional[Context] = None):
    """ChebyshevSemiIteration(M(level), scale, extra, steps).apply(b)."""
    ctx = ctx or default_context()
    n = ((1 << level) - 1) ** 2
    a = _Arg()
    out = np.zeros(n)
    _lib.check(ctx._L.oc_cheb_apply(ctx.h, level, C.c_double(scale),
                                    a.ptr(extra, n) if extra is not None else None, steps,
                                    a.ptr(b, n), C.c_void_p(out.ctypes.data)))
    return out


ASSEMBLE = {"mass": 0, "poisson": 1, "convdiff": 2, "partial_mass": 3, "lumped": 4}


def assemble9(what: str, level: int, eps: float = 0.1, obs=None) -> np.ndarray:
    """Host-side Q1 assembly (fem.cpp:142-180) into 9 coefficient arrays."""
    L = _lib.load()
    Grid(level)  # Grid: level out of range (grid.hpp:20)
    n = ((1 << level) - 1) ** 2
    out = np.zeros(n if what == "lumped" else 9 * n)
    o = np.ascontiguousarray(obs if obs is not None else [0.0, 1.0, 0.0, 1.0], dtype=np.float64)
    _lib.check(L.oc_assemble9(ASSEMBLE[what], level, C.c_double(eps),
                              C.c_void_p(o.ctypes.data), C.c_void_p(out.ctypes.data)))
    return out if what == "lumped" else out.reshape(9, n)


def assemble9_device(what: str, level: int, eps: float = 0.1, obs=None,
                     ctx: Optional[Context] = None) -> np.ndarray:
    """The same assembly run on the device (k_assembly.cu); what: mass,
    poisson, convdiff, partial_mass."""
    ctx = ctx or default_context()
    Grid(level)
    if what not in ("mass", "poisson", "convdiff", "partial_mass"):
        raise OptconInvalidArgument(f"assemble9_device: unsupported operator {what}")
    n = ((1 << level) - 1) ** 2
    out = np.zeros(9 * n)
    o = np.ascontiguousarray(obs if obs is not None else [0.0, 1.0, 0.0, 1.0], dtype=np.float64)
    _lib.check(ctx._L.oc_assemble9_device(ctx.h, ASSEMBLE[what], level, C.c_double(eps),
                                          C.c_void_p(o.ctypes.data), C.c_void_p(out.ctypes.data)))
    return out.reshape(9, n)
