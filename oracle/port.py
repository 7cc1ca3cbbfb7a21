"""numpy/scipy restatement of the reference hot path (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may use
this module, and only as the checker. Each function cites the reference
file:line it restates (paths under /root/reference/proj). It is pinned against
the reference itself (oracle/_ref, tests/test_port.py) and against the
committed golden fixtures. It also restates the 4-colour Gauss-Seidel variant
the GPU uses (``smoother="color4"``) so the device multigrid can be checked
against an independent implementation of exactly its algorithm.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp
import scipy.sparse.linalg as spla

# ---------------------------------------------------------------- assembly
_G = 0.57735026918962576
_Q = np.array([[-_G, -_G], [_G, -_G], [_G, _G], [-_G, _G]])
_LX = np.array([0, 1, 1, 0])
_LY = np.array([0, 0, 1, 1])


def _shape(xi, eta):
    return np.array([0.25 * (1 - xi) * (1 - eta), 0.25 * (1 + xi) * (1 - eta),
                     0.25 * (1 + xi) * (1 + eta), 0.25 * (1 - xi) * (1 + eta)])


def _grad(xi, eta):
    return np.array([[-0.25 * (1 - eta), -0.25 * (1 - xi)], [0.25 * (1 - eta), -0.25 * (1 + xi)],
                     [0.25 * (1 + eta), 0.25 * (1 + xi)], [-0.25 * (1 + eta), 0.25 * (1 - xi)]])


def element_mass(h):
    """fem.cpp:35-45"""
    m = np.zeros((4, 4))
    for q in _Q:
        N = _shape(*q)
        m += np.outer(N, N) * (h * h / 4.0)
    return m


def element_stiffness(h):
    """fem.cpp:47-59"""
    k = np.zeros((4, 4))
    s = 2.0 / h
    for q in _Q:
        G = _grad(*q)
        k += s * s * (G @ G.T) * (h * h / 4.0)
    return k


def wind(x1, x2):
    """default_wind, fem.cpp:164-169"""
    return 2.0 * x2 * (1.0 - x1 * x1), -2.0 * x1 * (1.0 - x2 * x2)


def element_convdiff_all(level, eps, supg=True):
    """fem.cpp:61-106 for every element at once: array (ne, ne, 4, 4)."""
    ne = 1 << level
    h = 1.0 / ne
    ex, ey = np.meshgrid(np.arange(ne), np.arange(ne))  # [ey, ex]
    x0, y0 = ex * h, ey * h
    a = np.broadcast_to(eps * element_stiffness(h), (ne, ne, 4, 4)).copy()
    wc = wind(x0 + 0.5 * h, y0 + 0.5 * h)
    wn = np.hypot(wc[0], wc[1])
    delta = np.zeros_like(wn)
    if supg:
        ok = wn > 1e-14
        pe = np.where(ok, wn * h / (2.0 * eps), 1.0)
        delta = np.where(ok, h / (2.0 * np.where(ok, wn, 1.0)) * np.maximum(0.0, 1.0 - 1.0 / pe), 0.0)
    s = 2.0 / h
    detj = h * h / 4.0
    for q in _Q:
        N = _shape(*q)
        G = _grad(*q)
        w0, w1 = wind(x0 + 0.5 * h * (q[0] + 1.0), y0 + 0.5 * h * (q[1] + 1.0))
        wg = s * (w0[..., None] * G[:, 0] + w1[..., None] * G[:, 1])  # (ne,ne,4)
        a += wg[..., None, :] * N[None, None, :, None] * detj
        a += delta[..., None, None] * wg[..., None, :] * wg[..., :, None] * detj
    return a


def assemble9(level, elem):
    """Scatter element matrices (fem.cpp:118-140): elem (4,4) or (ne,ne,4,4)."""
    ne = 1 << level
    nx = ne - 1
    n = nx * nx
    coef = np.zeros((9, n))
    E = np.asarray(elem)
    ex, ey = np.meshgrid(np.arange(ne), np.arange(ne))
    for i in range(4):
        gxi, gyi = ex + _LX[i], ey + _LY[i]
        for j in range(4):
            gxj, gyj = ex + _LX[j], ey + _LY[j]
            ok = (gxi >= 1) & (gxi <= nx) & (gyi >= 1) & (gyi <= nx) & \
                 (gxj >= 1) & (gxj <= nx) & (gyj >= 1) & (gyj <= nx)
            d = (gyj - gyi + 1) * 3 + (gxj - gxi + 1)
            row = (gyi - 1) * nx + (gxi - 1)
            val = E[..., i, j] if E.ndim == 4 else np.full(ex.shape, E[i, j])
            np.add.at(coef, (d[ok], row[ok]), val[ok])
    return coef


def assemble(what, level, eps=0.1, obs=None):
    h = 1.0 / (1 << level)
    if what == "mass":
        return assemble9(level, element_mass(h))
    if what == "poisson":
        return assemble9(level, element_stiffness(h))
    if what == "convdiff":
        return assemble9(level, element_convdiff_all(level, eps))
    if what == "partial_mass":
        ne = 1 << level
        ex, ey = np.meshgrid(np.arange(ne), np.arange(ne))
        tol = 1e-12  # grid.hpp:53-57
        inside = (ex * h >= obs[0] - tol) & ((ex + 1) * h <= obs[1] + tol) & \
                 (ey * h >= obs[2] - tol) & ((ey + 1) * h <= obs[3] + tol)
        E = np.where(inside[..., None, None], element_mass(h), 0.0)
        return assemble9(level, E)
    if what == "lumped":
        return assemble9(level, element_mass(h)).sum(axis=0)
    raise ValueError(what)


def to_csr(coef):
    n = coef.shape[1]
    nx = int(round(np.sqrt(n)))
    rows, cols, vals = [], [], []
    idx = np.arange(n)
    gx, gy = idx % nx, idx // nx
    for d in range(9):
        jx, jy = gx + d % 3 - 1, gy + d // 3 - 1
        ok = (jx >= 0) & (jx < nx) & (jy >= 0) & (jy < nx)
        rows.append(idx[ok]); cols.append((jy * nx + jx)[ok]); vals.append(coef[d][ok])
    return sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                         shape=(n, n))


def prolongation(fine_level):
    """bilinear_prolongation, multigrid.cpp:10-42."""
    nxf = (1 << fine_level) - 1
    nxc = (1 << (fine_level - 1)) - 1
    i = np.arange(1, nxf + 1)
    rows, cols, vals = [], [], []
    # 1D weights
    def s1(i):
        out = []
        if i % 2 == 0:
            out.append((i // 2, 1.0))
        else:
            if (i - 1) // 2 >= 1:
                out.append(((i - 1) // 2, 0.5))
            if (i + 1) // 2 <= nxc:
                out.append(((i + 1) // 2, 0.5))
        return out
    S = [s1(k) for k in i]
    P1 = np.zeros((nxf, nxc))
    for a, lst in enumerate(S):
        for c, w in lst:
            P1[a, c - 1] = w
    return sp.csr_matrix(np.kron(P1, P1))


# ---------------------------------------------------------------- multigrid
_SPLIT_CACHE = {}


def _split(A):
    key = id(A)
    hit = _SPLIT_CACHE.get(key)
    if hit is None or hit[0] is not A:
        DL = sp.tril(A, 0).tocsr()
        DU = sp.triu(A, 0).tocsr()
        hit = (A, DL, DU, sp.triu(A, 1).tocsr(), sp.tril(A, -1).tocsr())
        _SPLIT_CACHE[key] = hit
    return hit[1:]


def gs_lex(A, b, x, forward):
    """gauss_seidel_sweep (multigrid.cpp:44-66) via triangular solves:
    forward (D+L) x' = b - U x, backward (D+U) x' = b - L x."""
    DL, DU, Up, Lo = _split(A)
    if forward:
        return spla.spsolve_triangular(DL, b - Up @ x, lower=True)
    return spla.spsolve_triangular(DU, b - Lo @ x, lower=False)


def gs_color4(A, b, x, forward):
    """4-colour symmetric Gauss-Seidel (the GPU smoother): colour (gx&1)+2(gy&1),
    colours 0..3 forward, 3..0 backward; one Jacobi-style update per colour."""
    n = A.shape[0]
    nx = int(round(np.sqrt(n)))
    idx = np.arange(n)
    col = (idx % nx) % 2 + 2 * ((idx // nx) % 2)
    d = A.diagonal()
    x = x.copy()
    for c in (range(4) if forward else range(3, -1, -1)):
        m = col == c
        r = b[m] - (A[m] @ x) + d[m] * x[m]
        x[m] = r / d[m]
    return x


class MgHierarchy:
    """MgHierarchy (multigrid.cpp:75-157); smoother 'lex' (reference) or 'color4'."""

    def __init__(self, fine: sp.csr_matrix, level: int, rediscretize=None, smoother="lex"):
        if level < 3:
            raise ValueError("MgHierarchy: fine level must be >= 3")
        self.A = [sp.csr_matrix(fine)]
        self.P = []
        self.smoother = smoother
        rem = None
        if rediscretize is not None:
            rem = self.A[0] - rediscretize(level)
        for l in range(level, 2, -1):
            P = prolongation(l)
            R = P.T.tocsr()
            if rediscretize is not None:
                rem = (R @ (rem @ P)).tocsr()
                coarse = (rediscretize(l - 1) + rem).tocsr()
            else:
                coarse = (R @ (self.A[-1] @ P)).tocsr()
            self.P.append(P)
            self.A.append(coarse)
        self.lu = sla.lu_factor(self.A[-1].toarray())

    def depth(self):
        return len(self.P)

    def _sweep(self, A, b, x, forward):
        return gs_lex(A, b, x, forward) if self.smoother == "lex" else gs_color4(A, b, x, forward)

    def cycle(self, k, b, x, pre, post):
        if k + 1 == len(self.A):
            return sla.lu_solve(self.lu, b)
        A = self.A[k]
        for _ in range(pre):
            x = self._sweep(A, b, x, True)
        r = b - A @ x
        rc = self.P[k].T @ r
        ec = self.cycle(k + 1, rc, np.zeros(rc.size), pre, post)
        x = x + self.P[k] @ ec
        for _ in range(post):
            x = self._sweep(A, b, x, False)
        return x

    def solve(self, b, cycles=3, pre=5, post=5):
        x = np.zeros(b.size)
        prev = np.linalg.norm(b)
        if prev == 0.0:
            return x
        for _ in range(cycles):
            x = self.cycle(0, b, x, pre, post)
            res = np.linalg.norm(b - self.A[0] @ x)
            if res > 10.0 * prev:
                raise RuntimeError("MgHierarchy::solve: residual growth, cycle diverged")
            prev = res
        return x


def chebyshev(M: sp.csr_matrix, scale, extra, steps, b):
    """ChebyshevSemiIteration (chebyshev.cpp:9-75)."""
    d = M.diagonal()
    inv = 1.0 / (scale * d + extra)
    lmin, lmax = 0.25, 2.25
    omega = 2.0 / (lmin + lmax)
    rho = (lmax - lmin) / (lmax + lmin)
    g = omega * inv * b
    prev = np.zeros_like(b)
    cur = g.copy()
    w = 1.0
    for step in range(2, steps + 1):
        w = 1.0 / (1.0 - 0.5 * rho * rho) if step == 2 else 1.0 / (1.0 - 0.25 * rho * rho * w)
        az = M @ cur
        if scale != 1.0:
            az = scale * az
        az = az + extra * cur
        s_cur = cur - omega * inv * az
        nxt = w * (s_cur + g - prev) + prev
        prev, cur = cur, nxt
    return cur


# ---------------------------------------------------------------- Krylov
def gmres(A, P, b, tol=1e-10, maxit=200):
    """krylov.cpp:133-212 (full, right-preconditioned, true residual each step)."""
    n = b.size
    bnorm = np.linalg.norm(b)
    x = np.zeros(n)
    rep = dict(iterations=0, relative_residual=0.0, converged=False)
    if bnorm == 0.0:
        rep["converged"] = True
        return x, rep
    V = [b / bnorm]
    Z, H, cs, sn, g = [], [], [], [], [bnorm]
    for j in range(maxit):
        Z.append(P(V[j]))
        w = A(Z[-1])
        h = np.zeros(j + 2)
        for i in range(j + 1):
            h[i] = w @ V[i]
            w = w - h[i] * V[i]
        hn = np.linalg.norm(w)
        h[j + 1] = hn
        for i in range(j):
            t = cs[i] * h[i] + sn[i] * h[i + 1]
            h[i + 1] = -sn[i] * h[i] + cs[i] * h[i + 1]
            h[i] = t
        r = np.hypot(h[j], hn)
        if r == 0.0:
            break
        cs.append(h[j] / r)
        sn.append(hn / r)
        h[j] = r
        g.append(-sn[-1] * g[-1])
        g[j] *= cs[-1]
        H.append(h)
        if hn > 1e-300:
            V.append(w / hn)
        m = j + 1
        y = np.zeros(m)
        for i in range(m - 1, -1, -1):
            s = g[i] - sum(H[k][i] * y[k] for k in range(i + 1, m))
            y[i] = s / H[i][i]
        x = sum(y[i] * Z[i] for i in range(m))
        rep["iterations"] = m
        rep["relative_residual"] = np.linalg.norm(b - A(x)) / bnorm
        if rep["relative_residual"] <= tol:
            rep["converged"] = True
            return x, rep
        if hn <= 1e-300:
            return x, rep
    return x, rep


def minres(A, P, b, tol=1e-10, maxit=200):
    """krylov.cpp:37-131."""
    n = b.size
    x = np.zeros(n)
    rep = dict(iterations=0, relative_residual=0.0, converged=False, breakdown=False)
    bnorm = np.linalg.norm(b)
    if bnorm == 0.0:
        rep["converged"] = True
        return x, rep
    v_prev, v = np.zeros(n), b.copy()
    z = P(v)
    gsq = z @ v
    if not gsq > 0.0:
        rep.update(breakdown=True, relative_residual=1.0)
        return x, rep
    gamma, gamma_prev, eta = np.sqrt(gsq), 1.0, np.sqrt(gsq)
    c_prev = c = 1.0
    s_prev = s = 0.0
    w_prev, w = np.zeros(n), np.zeros(n)
    for j in range(1, maxit + 1):
        z = z * (1.0 / gamma)
        az = A(z)
        delta = az @ z
        v_next = az - (delta / gamma) * v
        if j > 1:
            v_next = v_next - (gamma / gamma_prev) * v_prev
        z_next = P(v_next)
        gn_sq = z_next @ v_next
        if gn_sq < 0.0:
            rep.update(breakdown=True, iterations=j,
                       relative_residual=np.linalg.norm(b - A(x)) / bnorm)
            return x, rep
        gn = np.sqrt(gn_sq)
        a0 = c * delta - c_prev * s * gamma
        a1 = np.sqrt(a0 * a0 + gn * gn)
        a2 = s * delta + c_prev * c * gamma
        a3 = s_prev * gamma
        if a1 == 0.0:
            rr = np.linalg.norm(b - A(x)) / bnorm
            rep.update(iterations=j, relative_residual=rr, converged=rr <= tol)
            return x, rep
        c_next, s_next = a0 / a1, gn / a1
        w_next = (z - a3 * w_prev - a2 * w) * (1.0 / a1)
        x = x + (c_next * eta) * w_next
        eta = -s_next * eta
        v_prev, v, z = v, v_next, z_next
        gamma_prev, gamma = gamma, gn
        w_prev, w = w, w_next
        c_prev, c, s_prev, s = c, c_next, s, s_next
        rep["iterations"] = j
        rep["relative_residual"] = np.linalg.norm(b - A(x)) / bnorm
        if rep["relative_residual"] <= tol:
            rep["converged"] = True
            return x, rep
        if gamma == 0.0:
            break
    return x, rep


# ---------------------------------------------------------------- QP + IPM
@dataclass
class Qp:
    """QpProblem (qp.hpp:53-77) built as in build_qp (qp.cpp:123-174)."""

    level: int
    pde: str
    alpha: float
    beta: float
    y_d: np.ndarray
    u_a: np.ndarray
    u_b: np.ndarray
    y_a: Optional[np.ndarray] = None
    y_b: Optional[np.ndarray] = None
    obs: Optional[tuple] = None
    eps: float = 0.1
    f_nodal: Optional[np.ndarray] = None
    smoother: str = "lex"
    M: sp.csr_matrix = field(init=False)

    def __post_init__(self):
        l = self.level
        self.n = ((1 << l) - 1) ** 2
        self.M = to_csr(assemble("mass", l))
        self.lumped = np.asarray(self.M.sum(axis=1)).ravel()
        if self.pde == "poisson":
            self.L = to_csr(assemble("poisson", l))
            self.assembler = None
        else:
            self.L = to_csr(assemble("convdiff", l, self.eps))
            eps = self.eps
            self.assembler = lambda lv: to_csr(assemble("convdiff", lv, eps))
        self.LT = self.L.T.tocsr()
        self.partial = self.obs is not None
        self.Mobs = to_csr(assemble("partial_mass", l, obs=self.obs)) if self.partial else self.M
        fn = np.zeros(self.n) if self.f_nodal is None else self.f_nodal
        self.f = self.M @ fn
        n = self.n
        ua = np.broadcast_to(self.u_a, (n,)).astype(float)
        ub = np.broadcast_to(self.u_b, (n,)).astype(float)
        self.z_a = np.r_[np.maximum(ua, 0.0), -np.minimum(ub, 0.0)]
        self.z_b = np.r_[np.maximum(ub, 0.0), -np.minimum(ua, 0.0)]
        pin = self.z_b - self.z_a < 1e-12
        self.z_b[pin] = self.z_a[pin] + 1e-12
        if self.y_a is not None:
            self.y_a = np.broadcast_to(self.y_a, (n,)).astype(float)
            self.y_b = np.broadcast_to(self.y_b, (n,)).astype(float)
        self.dM = self.M.diagonal()

    # steady_matvecs (ipm.cpp:347-374)
    def hy(self, v):
        return self.Mobs @ v

    def hz(self, z):
        n = self.n
        m = self.M @ (z[:n] - z[n:])
        return np.r_[self.alpha * m, self.alpha * (-m)]

    def k(self, y):
        return self.L @ y

    def kt(self, p):
        return self.LT @ p

    def b(self, z):
        n = self.n
        return self.M @ (z[:n] - z[n:])

    def bt(self, p):
        mp = self.M @ p
        return np.r_[mp, -mp]

    def beta_grad(self):
        return np.r_[self.beta * self.lumped, self.beta * self.lumped]

    def objective(self, y, z):
        """qp.cpp:112-121"""
        n = self.n
        d = y - self.y_d
        val = 0.5 * (d @ (self.Mobs @ d))
        val += 0.5 * self.alpha * (z @ np.r_[self.M @ (z[:n] - z[n:]), -(self.M @ (z[:n] - z[n:]))])
        return val + self.beta * (self.lumped @ (z[:n] + z[n:]))

    def kkt(self, ty, tw, tv, x):
        """make_saddle_operator (ipm.cpp:237-268)."""
        n = self.n
        y, z, p = x[:n], x[n:3 * n], x[3 * n:]
        ry = self.hy(y) + ty * y + self.kt(p)
        rz = self.hz(z) + np.r_[tw, tv] * z - self.bt(p)
        rp = self.k(y) - self.b(z)
        return np.r_[ry, rz, rp]

    # ------------------------------------------------ preconditioners
    def mg_opts(self):
        return dict(rediscretize=self.assembler, smoother=self.smoother)

    def bracket(self, tw, tv):
        """matching_bracket (precond.cpp:55-72)."""
        d = self.dM
        s = 1.0 / tw + 1.0 / tv
        return np.maximum(d * d * s / (self.alpha * d * s + 1.0), 0.0)

    def setup(self, ty, tw, tv, kind):
        self.th = (ty, tw, tv)
        d = self.dM
        self.a2 = self.alpha * d + tw
        self.b2 = -self.alpha * d
        self.c2 = self.alpha * d + tv
        l = self.level
        if kind == "ppi":
            br = self.bracket(tw, tv)
            self.mgL = MgHierarchy(self.L, l, **self.mg_opts())
            left = (self.LT + self.Mobs + sp.diags(ty)).tocsr()
            tasm = None if self.assembler is None else (lambda lv: self.assembler(lv).T.tocsr())
            self.mg_left = MgHierarchy(left, l, rediscretize=tasm, smoother=self.smoother)
            self.mg_right = MgHierarchy((self.L + sp.diags(br)).tocsr(), l, **self.mg_opts())
        else:
            mhat = np.sqrt(self.bracket(tw, tv)) * np.sqrt(d + ty)
            F = (self.L + sp.diags(mhat)).tocsr()
            self.mgF = MgHierarchy(F, l, **self.mg_opts())
            tasm = None if self.assembler is None else (lambda lv: self.assembler(lv).T.tocsr())
            self.mgFT = MgHierarchy(F.T.tocsr(), l, rediscretize=tasm, smoother=self.smoother)

    def two_by_two(self, r1, r2):
        """block_2x2_inverse_apply (precond.cpp:37-53)."""
        a, b, c = self.a2, self.b2, self.c2
        schur = c - b * b / a
        x2 = (r2 - b * r1 / a) / schur
        x1 = (r1 - b * x2) / a
        return x1, x2

    def schur(self, r, cyc=(3, 5, 5)):
        """SchurApprox::apply_inverse (precond.cpp:130-136)."""
        t1 = self.mgF.solve(r, *cyc)
        t2 = self.Mobs @ t1 + self.th[0] * t1
        return self.mgFT.solve(t2, *cyc)

    def precond(self, kind, r, cheb_steps=20, cyc=(3, 5, 5)):
        n = self.n
        ry, rw, rv, rp = r[:n], r[n:2 * n], r[2 * n:3 * n], r[3 * n:]
        ty = self.th[0]
        vw, vv = self.two_by_two(rw, rv)
        if kind == "ppi":
            rhs1 = self.M @ (vw - vv) + rp
            v1 = self.mgL.solve(rhs1, *cyc)
            t = self.Mobs @ v1 + (ty * v1 - ry)
            v3 = self.mg_right.solve(self.L @ self.mg_left.solve(t, *cyc), *cyc)
            return np.r_[v1, vw, vv, v3]
        vy = chebyshev(self.Mobs, 1.0, ty, cheb_steps, ry)
        if kind == "pt":
            t = self.L @ vy + (-(self.M @ vw) + self.M @ vv - rp)
            vp = self.schur(t, cyc)
        else:
            vp = self.schur(rp, cyc)
        return np.r_[vy, vw, vv, vp]


def ipm_solve(qp: Qp, sigma=0.2, solver="gmres-pt", alpha0=0.995, eps=1e-6, mu0=1.0,
              max_iterations=100, linear_tol=1e-10, linear_maxit=200, cheb_steps=20,
              mg=(3, 5, 5), max_newton=None):
    """ipm_solve (ipm.cpp:270-341) over the steady model (ipm.cpp:388-470).
    max_newton bounds the number of IPM iterations (CPU-baseline sampling)."""
    n = qp.n
    sb = qp.y_a is not None
    y = qp.y_d.copy()
    if sb:
        delta = 1e-2 * (qp.y_b - qp.y_a)
        y = np.minimum(np.maximum(y, qp.y_a + delta), qp.y_b - delta)
        lya, lyb = np.ones(n), np.ones(n)
    z = 0.5 * (qp.z_a + qp.z_b)
    p = np.zeros(n)
    lza, lzb = np.ones(2 * n), np.ones(2 * n)
    bg = qp.beta_grad()

    def residuals(mu):
        xp = qp.k(y) - qp.b(z) - qp.f
        xdy = qp.hy(y - qp.y_d) + qp.kt(p)
        if sb:
            xdy = xdy - lya + lyb
        xdz = qp.hz(z) + bg - qp.bt(p) - lza + lzb
        xc = []
        if sb:
            xc += [(y - qp.y_a) * lya - mu, (qp.y_b - y) * lyb - mu]
        xc += [(z - qp.z_a) * lza - mu, (qp.z_b - z) * lzb - mu]
        xd = np.r_[xdy, xdz]
        xc = np.concatenate(xc)
        return (np.linalg.norm(xp) / np.sqrt(xp.size), np.linalg.norm(xd) / np.sqrt(xd.size),
                np.linalg.norm(xc) / np.sqrt(xc.size))

    state_mu = mu0
    norms = residuals(mu0)
    records = [dict(k=0, mu=mu0, norms=norms, lin_iters=0)]
    k = 0
    mu = mu0
    total = 0
    kind = {"gmres-pt": "pt", "minres-pd": "pd", "gmres-ppi": "ppi"}[solver]

    def conv():
        return norms[0] <= eps and norms[1] <= eps and norms[2] <= eps and state_mu <= eps

    while not conv() and k < max_iterations and (max_newton is None or k < max_newton):
        mu = sigma * mu
        tw = lza[:n] / (z[:n] - qp.z_a[:n]) + lzb[:n] / (qp.z_b[:n] - z[:n])
        tv = lza[n:] / (z[n:] - qp.z_a[n:]) + lzb[n:] / (qp.z_b[n:] - z[n:])
        ty = lya / (y - qp.y_a) + lyb / (qp.y_b - y) if sb else np.zeros(n)
        r1 = qp.hy(y - qp.y_d) + qp.kt(p)
        if sb:
            r1 = r1 - mu / (y - qp.y_a) + mu / (qp.y_b - y)
        r2 = qp.hz(z) + bg - qp.bt(p) - mu / (z - qp.z_a) + mu / (qp.z_b - z)
        r3 = qp.k(y) - qp.b(z) - qp.f
        rhs = -np.r_[r1, r2, r3]
        qp.setup(ty, tw, tv, kind)
        A = lambda v: qp.kkt(ty, tw, tv, v)  # noqa: E731
        P = lambda v: qp.precond(kind, v, cheb_steps, mg)  # noqa: E731
        x, rep = (minres if kind == "pd" else gmres)(A, P, rhs, linear_tol, linear_maxit)
        dy, dz, dp = x[:n], x[n:3 * n], x[3 * n:]
        lo, hi = z - qp.z_a, qp.z_b - z
        dlza = -lza / lo * dz - lza + mu / lo
        dlzb = lzb / hi * dz - lzb + mu / hi

        def box(xv, dx, a, b):
            r = np.inf
            m = dx < 0
            if m.any():
                r = min(r, np.min((a[m] - xv[m]) / dx[m]))
            m = dx > 0
            if m.any():
                r = min(r, np.min((b[m] - xv[m]) / dx[m]))
            return r

        def zero(lam, dl):
            m = dl < 0
            return np.min(-lam[m] / dl[m]) if m.any() else np.inf

        rp = box(z, dz, qp.z_a, qp.z_b)
        rd = min(zero(lza, dlza), zero(lzb, dlzb))
        if sb:
            ylo, yhi = y - qp.y_a, qp.y_b - y
            dlya = -lya / ylo * dy - lya + mu / ylo
            dlyb = lyb / yhi * dy - lyb + mu / yhi
            rp = min(rp, box(y, dy, qp.y_a, qp.y_b))
            rd = min(rd, zero(lya, dlya), zero(lyb, dlyb))
        ap, ad = min(1.0, alpha0 * rp), min(1.0, alpha0 * rd)
        y = y + ap * dy
        z = z + ap * dz
        p = p + ad * dp
        lza = lza + ad * dlza
        lzb = lzb + ad * dlzb
        if sb:
            lya = lya + ad * dlya
            lyb = lyb + ad * dlyb
        state_mu = mu
        k += 1
        norms = residuals(mu)
        total += rep["iterations"]
        records.append(dict(k=k, mu=mu, norms=norms, lin_iters=rep["iterations"],
                            relres=rep["relative_residual"]))
    u = z[:n] - z[n:]
    return dict(y=y, z=z, p=p, u=u, nli=k, av_li=total / k if k else 0.0, total_lin=total,
                converged=conv(), objective=qp.objective(y, z), records=records, mu=state_mu)
