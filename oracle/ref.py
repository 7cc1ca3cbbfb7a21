"""ctypes driver for the reference library built by oracle/Makefile.

TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's
CPU-baseline leg (``--impl reference`` / ``cpu_baseline``) may import this
module. It loads ``oracle/_ref/liboptcon_ref.so`` — the reference optcon
sources from /root/reference/proj/src compiled unmodified plus our harness
(oracle/ref_harness.cpp) — and exposes the reference solver on numpy arrays.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# OPTCON_REF_LIB selects a rounding-variant build of the same sources (Makefile EXTRA)
LIB_PATH = os.environ.get("OPTCON_REF_LIB") or os.path.join(_HERE, "_ref", "liboptcon_ref.so")

_dp = C.POINTER(C.c_double)


class ProblemDesc(C.Structure):
    _fields_ = [
        ("pde", C.c_int), ("level", C.c_int), ("eps", C.c_double), ("tau", C.c_double),
        ("horizon", C.c_double), ("quadrature", C.c_int), ("alpha", C.c_double),
        ("beta", C.c_double), ("y_d", _dp), ("y_d_len", C.c_longlong), ("f", _dp),
        ("u_a", _dp), ("u_b", _dp), ("y_a", _dp), ("y_b", _dp), ("has_obs", C.c_int),
        ("obs", C.c_double * 4),
    ]


class Params(C.Structure):
    _fields_ = [
        ("alpha0", C.c_double), ("sigma", C.c_double), ("eps_p", C.c_double),
        ("eps_d", C.c_double), ("eps_c", C.c_double), ("mu0", C.c_double),
        ("max_iterations", C.c_int), ("linear_tol", C.c_double), ("linear_maxit", C.c_int),
        ("cheb_steps", C.c_int), ("mg_cycles", C.c_int), ("mg_pre", C.c_int),
        ("mg_post", C.c_int), ("solver", C.c_int),
    ]


class Record(C.Structure):
    _fields_ = [
        ("k", C.c_int), ("mu", C.c_double), ("norm_xp", C.c_double), ("norm_xd", C.c_double),
        ("norm_xc", C.c_double), ("lin_iters", C.c_int), ("lin_relres", C.c_double),
        ("lin_converged", C.c_int), ("newton_seconds", C.c_double),
    ]


class Result(C.Structure):
    _fields_ = [
        ("y", _dp), ("z", _dp), ("p", _dp), ("lam_ya", _dp), ("lam_yb", _dp),
        ("lam_za", _dp), ("lam_zb", _dp), ("u", _dp), ("records", C.POINTER(Record)),
        ("records_cap", C.c_int), ("n_records", C.c_int), ("nli", C.c_int),
        ("converged", C.c_int), ("av_li", C.c_double), ("mu", C.c_double),
        ("objective", C.c_double), ("sparsity_pct", C.c_double), ("l1", C.c_double),
        ("nodal_sparsity_pct", C.c_double), ("total_lin", C.c_longlong),
        ("newton_seconds", C.c_double), ("solve_seconds", C.c_double),
    ]


SOLVERS = {"gmres-pt": 0, "minres-pd": 1, "gmres-ppi": 2, "dense": 3, "heat-minres-pd": 10}
PDES = {"poisson": 0, "convdiff": 1, "heat": 2}


class RefError(RuntimeError):
    pass


class RefInvalidArgument(RefError, ValueError):
    pass


_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise RefError(f"reference oracle not built: {LIB_PATH} (run make -C oracle)")
        L = C.CDLL(LIB_PATH)
        L.ref_last_error.restype = C.c_char_p
        L.ref_problem_create.restype = C.c_void_p
        L.ref_problem_create.argtypes = [C.POINTER(ProblemDesc)]
        L.ref_problem_destroy.argtypes = [C.c_void_p]
        L.ref_mg_create.restype = C.c_void_p
        L.ref_mg_create.argtypes = [C.c_int, _dp, C.c_int, C.c_double, C.c_int]
        L.ref_mg_destroy.argtypes = [C.c_void_p]
        for name in ["ref_problem_sizes", "ref_ipm_solve", "ref_kkt_apply", "ref_precond_setup",
                     "ref_precond_apply", "ref_schur_apply", "ref_time_applies", "ref_objective",
                     "ref_ipm_pieces", "ref_assemble9", "ref_mg_solve", "ref_mg_depth",
                     "ref_mg_level_matrix", "ref_gs_sweep", "ref_cheb_apply", "ref_krylov_9diag",
                     "ref_newton_sample_prepare", "ref_newton_sample_run"]:
            getattr(L, name).restype = C.c_int
        _lib = L
    return _lib


def _check(rc: int):
    if rc != 0:
        msg = lib().ref_last_error().decode()
        if rc == 1:
            raise RefInvalidArgument(msg)
        raise RefError(msg)


def _ptr(a: np.ndarray | None):
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


def params(solver="gmres-pt", **kw) -> Params:
    p = Params(alpha0=0.995, sigma=0.2, eps_p=1e-6, eps_d=1e-6, eps_c=1e-6, mu0=1.0,
               max_iterations=100, linear_tol=1e-10, linear_maxit=200, cheb_steps=20,
               mg_cycles=3, mg_pre=5, mg_post=5, solver=SOLVERS[solver])
    for k, v in kw.items():
        setattr(p, k, v)
    return p


@dataclass
class RefSolve:
    y: np.ndarray
    z: np.ndarray
    p: np.ndarray
    lam_za: np.ndarray
    lam_zb: np.ndarray
    lam_ya: np.ndarray | None
    lam_yb: np.ndarray | None
    u: np.ndarray
    records: list = field(default_factory=list)
    nli: int = 0
    converged: bool = False
    av_li: float = 0.0
    mu: float = 0.0
    objective: float = 0.0
    sparsity_pct: float = 0.0
    l1: float = 0.0
    nodal_sparsity_pct: float = 0.0
    total_lin: int = 0
    newton_seconds: float = 0.0
    solve_seconds: float = 0.0


class RefProblem:
    """Reference ControlProblem -> build_qp/assemble_spacetime -> IpmModel."""

    def __init__(self, pde="poisson", level=6, alpha=1e-2, beta=1e-2, y_d=None, u_a=-2.0,
                 u_b=1.5, y_a=None, y_b=None, obs=None, eps=1e-1, tau=0.04, horizon=1.0,
                 quadrature=0, f=None):
        nx = (1 << level) - 1
        n = nx * nx
        self._keep = []

        def arr(v, size):
            if v is None:
                return None
            a = np.ascontiguousarray(np.broadcast_to(np.asarray(v, dtype=np.float64), (size,)))
            a = a.copy()
            self._keep.append(a)
            return a

        yd = np.ascontiguousarray(np.asarray(y_d, dtype=np.float64))
        self._keep.append(yd)
        d = ProblemDesc()
        d.pde = PDES[pde]
        d.level = level
        d.eps = eps
        d.tau = tau
        d.horizon = horizon
        d.quadrature = quadrature
        d.alpha = alpha
        d.beta = beta
        d.y_d = _ptr(yd)
        d.y_d_len = yd.size
        d.f = _ptr(arr(f, n))
        d.u_a = _ptr(arr(u_a, n))
        d.u_b = _ptr(arr(u_b, n))
        d.y_a = _ptr(arr(y_a, n))
        d.y_b = _ptr(arr(y_b, n))
        if obs is not None:
            d.has_obs = 1
            for i in range(4):
                d.obs[i] = obs[i]
        self.h = lib().ref_problem_create(C.byref(d))
        if not self.h:
            msg = lib().ref_last_error().decode()
            raise RefInvalidArgument(msg) if "must" in msg or "mismatch" in msg else RefError(msg)
        n_, nt, sb = C.c_int(), C.c_int(), C.c_int()
        _check(lib().ref_problem_sizes(C.c_void_p(self.h), C.byref(n_), C.byref(nt), C.byref(sb)))
        self.n, self.nt, self.has_state_bounds = n_.value, nt.value, bool(sb.value)
        self.ny = self.n * self.nt
        self.level = level

    def __del__(self):
        h = getattr(self, "h", None)
        if h and _lib is not None:
            _lib.ref_problem_destroy(C.c_void_p(h))
            self.h = None

    def solve(self, solver="gmres-pt", **kw) -> RefSolve:
        p = params(solver, **kw)
        ny = self.ny
        out = RefSolve(y=np.zeros(ny), z=np.zeros(2 * ny), p=np.zeros(ny),
                       lam_za=np.zeros(2 * ny), lam_zb=np.zeros(2 * ny),
                       lam_ya=np.zeros(ny) if self.has_state_bounds else None,
                       lam_yb=np.zeros(ny) if self.has_state_bounds else None,
                       u=np.zeros(ny))
        cap = 256
        recs = (Record * cap)()
        r = Result(y=_ptr(out.y), z=_ptr(out.z), p=_ptr(out.p), lam_ya=_ptr(out.lam_ya),
                   lam_yb=_ptr(out.lam_yb), lam_za=_ptr(out.lam_za), lam_zb=_ptr(out.lam_zb),
                   u=_ptr(out.u), records=C.cast(recs, C.POINTER(Record)), records_cap=cap)
        _check(lib().ref_ipm_solve(C.c_void_p(self.h), C.byref(p), C.byref(r)))
        out.records = [dict(k=recs[i].k, mu=recs[i].mu, norm_xp=recs[i].norm_xp,
                            norm_xd=recs[i].norm_xd, norm_xc=recs[i].norm_xc,
                            lin_iters=recs[i].lin_iters, lin_relres=recs[i].lin_relres,
                            lin_converged=bool(recs[i].lin_converged),
                            newton_seconds=recs[i].newton_seconds)
                       for i in range(min(r.n_records, cap))]
        for k in ["nli", "av_li", "mu", "objective", "sparsity_pct", "l1", "nodal_sparsity_pct",
                  "total_lin", "newton_seconds", "solve_seconds"]:
            setattr(out, k, getattr(r, k))
        out.converged = bool(r.converged)
        return out

    def kkt_apply(self, theta_y, theta_w, theta_v, x):
        out = np.zeros(4 * self.ny)
        args = [np.ascontiguousarray(a, dtype=np.float64) for a in (theta_y, theta_w, theta_v, x)]
        _check(lib().ref_kkt_apply(C.c_void_p(self.h), *[_ptr(a) for a in args], _ptr(out)))
        return out

    def precond_setup(self, theta_y, theta_w, theta_v, **kw):
        p = params("gmres-pt", **kw)
        args = [np.ascontiguousarray(a, dtype=np.float64) for a in (theta_y, theta_w, theta_v)]
        _check(lib().ref_precond_setup(C.c_void_p(self.h), *[_ptr(a) for a in args], C.byref(p)))

    def newton_sample_prepare(self, solver="gmres-pt", **kw) -> float:
        """Form the first IPM Newton system with the reference's ipm_solve and set
        up its preconditioner; returns the setup wall seconds."""
        p = params(solver, **kw)
        t = C.c_double()
        _check(lib().ref_newton_sample_prepare(C.c_void_p(self.h), C.byref(p), C.byref(t)))
        return t.value

    def newton_sample_run(self, kind, method, maxit, tol=1e-10):
        """The reference's gmres/minres on the prepared Newton system, at most
        `maxit` iterations: (iterations, relative residual, wall seconds)."""
        kinds = {"pd": 0, "pt": 1, "ppi": 2, "heat-pt": 3, "heat-pd": 4}
        it, rr, t = C.c_int(), C.c_double(), C.c_double()
        _check(lib().ref_newton_sample_run(C.c_void_p(self.h), kinds[kind],
                                           {"gmres": 0, "minres": 1}[method], C.c_double(tol),
                                           int(maxit), C.byref(it), C.byref(rr), C.byref(t)))
        return it.value, rr.value, t.value

    def precond_apply(self, kind, r):
        kinds = {"pd": 0, "pt": 1, "ppi": 2, "heat-pt": 3, "heat-pd": 4}
        r = np.ascontiguousarray(r, dtype=np.float64)
        out = np.zeros_like(r)
        _check(lib().ref_precond_apply(C.c_void_p(self.h), kinds[kind], _ptr(r), _ptr(out)))
        return out

    def schur_apply(self, r):
        r = np.ascontiguousarray(r, dtype=np.float64)
        out = np.zeros_like(r)
        _check(lib().ref_schur_apply(C.c_void_p(self.h), _ptr(r), _ptr(out)))
        return out

    def time_applies(self, kind, reps, x):
        kinds = {"pd": 0, "pt": 1, "ppi": 2, "heat-pt": 3, "heat-pd": 4}
        a, b = C.c_double(), C.c_double()
        x = np.ascontiguousarray(x, dtype=np.float64)
        _check(lib().ref_time_applies(C.c_void_p(self.h), kinds[kind], reps, _ptr(x),
                                      C.byref(a), C.byref(b)))
        return a.value, b.value

    def objective(self, y, z):
        o = C.c_double()
        y = np.ascontiguousarray(y, dtype=np.float64)
        z = np.ascontiguousarray(z, dtype=np.float64)
        _check(lib().ref_objective(C.c_void_p(self.h), _ptr(y), _ptr(z), C.byref(o)))
        return o.value

    def ipm_pieces(self, y, z, p, lam_za, lam_zb, lam_ya=None, lam_yb=None, mu_state=1.0,
                   mu_rhs=0.2):
        ny = self.ny
        th = [np.zeros(ny) for _ in range(3)]
        r1, r2, r3 = np.zeros(ny), np.zeros(2 * ny), np.zeros(ny)
        norms = np.zeros(3)
        args = [np.ascontiguousarray(a, dtype=np.float64) if a is not None else None
                for a in (y, z, p, lam_ya, lam_yb, lam_za, lam_zb)]
        _check(lib().ref_ipm_pieces(C.c_void_p(self.h), *[_ptr(a) for a in args],
                                    C.c_double(mu_state), C.c_double(mu_rhs),
                                    *[_ptr(t) for t in th], _ptr(r1), _ptr(r2), _ptr(r3),
                                    _ptr(norms)))
        return dict(theta_y=th[0], theta_w=th[1], theta_v=th[2], r1=r1, r2=r2, r3=r3,
                    norms=norms)


ASSEMBLE = {"mass": 0, "poisson": 1, "convdiff": 2, "partial_mass": 3, "lumped": 4}


def assemble9(what: str, level: int, eps: float = 0.1, obs=None) -> np.ndarray:
    nx = (1 << level) - 1
    n = nx * nx
    out = np.zeros(n if what == "lumped" else 9 * n)
    o = np.ascontiguousarray(obs if obs is not None else [0, 1, 0, 1], dtype=np.float64)
    _check(lib().ref_assemble9(ASSEMBLE[what], level, C.c_double(eps), _ptr(o), _ptr(out)))
    return out if what == "lumped" else out.reshape(9, n)


class RefMg:
    def __init__(self, level, coef9, rediscretize_convdiff=False, eps=0.1, transpose_base=False):
        self.level = level
        c = np.ascontiguousarray(coef9, dtype=np.float64).reshape(-1)
        self.h = lib().ref_mg_create(level, _ptr(c), int(rediscretize_convdiff), C.c_double(eps),
                                     int(transpose_base))
        if not self.h:
            raise RefError(lib().ref_last_error().decode())
        self.n = ((1 << level) - 1) ** 2

    def __del__(self):
        h = getattr(self, "h", None)
        if h and _lib is not None:
            _lib.ref_mg_destroy(C.c_void_p(h))

    def solve(self, rhs, cycles=3, pre=5, post=5):
        rhs = np.ascontiguousarray(rhs, dtype=np.float64)
        out = np.zeros_like(rhs)
        _check(lib().ref_mg_solve(C.c_void_p(self.h), _ptr(rhs), cycles, pre, post, _ptr(out)))
        return out

    def depth(self):
        return lib().ref_mg_depth(C.c_void_p(self.h))

    def level_matrix(self, k):
        nx = (1 << (self.level - k)) - 1
        out = np.zeros(9 * nx * nx)
        _check(lib().ref_mg_level_matrix(C.c_void_p(self.h), k, _ptr(out)))
        return out.reshape(9, nx * nx)


def gs_sweep(level, coef9, b, x, forward=True):
    c = np.ascontiguousarray(coef9, dtype=np.float64).reshape(-1)
    b = np.ascontiguousarray(b, dtype=np.float64)
    x = np.array(x, dtype=np.float64, copy=True)
    _check(lib().ref_gs_sweep(level, _ptr(c), _ptr(b), _ptr(x), int(forward)))
    return x


def cheb_apply(level, scale, extra, steps, b):
    b = np.ascontiguousarray(b, dtype=np.float64)
    e = None if extra is None else np.ascontiguousarray(extra, dtype=np.float64)
    out = np.zeros_like(b)
    _check(lib().ref_cheb_apply(level, C.c_double(scale), _ptr(e), steps, _ptr(b), _ptr(out)))
    return out
