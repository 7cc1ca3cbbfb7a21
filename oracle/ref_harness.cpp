// C harness over the reference optcon library (TEST INFRASTRUCTURE ONLY).
//
// This file is our own code. It links the reference sources compiled in place
// from /root/reference/proj/src (see oracle/Makefile) and exposes a C ABI so the
// Python tests and bench.py's CPU-baseline leg can drive the reference on the
// same seeded inputs the GPU path receives. It mirrors the reference's own
// entry pattern (tests/acceptance/acceptance_main.cpp:65-89: ControlProblem ->
// build_qp -> make_steady_model -> ipm_solve) and times newton_solve by
// wrapping the public IpmModel::newton_solve std::function (ipm.hpp:88-90).
#include "ref_harness.h"

#include "optcon/chebyshev.hpp"
#include "optcon/fem.hpp"
#include "optcon/ipm.hpp"
#include "optcon/krylov.hpp"
#include "optcon/multigrid.hpp"
#include "optcon/precond.hpp"
#include "optcon/qp.hpp"
#include "optcon/timedep.hpp"

#include <chrono>
#include <cmath>
#include <cstring>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>

using namespace optcon;

namespace {

thread_local std::string g_err;

template <typename F>
int guarded(F&& f)
{
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::runtime_error& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 3;
    }
}

double now_s()
{
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch())
        .count();
}

Vector from_ptr(const double* p, std::size_t n) { return Vector(p, p + n); }

void to_ptr(const Vector& v, double* p)
{
    if (p) std::memcpy(p, v.data(), v.size() * sizeof(double));
}

// CSR <-> 9 coefficient arrays in the order SW,S,SE,W,C,E,NW,N,NE (= ascending
// column order of a lexicographic 9-point row, grid.hpp:31-36).
void csr_to_9(const SparseMatrix& A, int level, double* coef)
{
    const Grid g(level);
    const std::int32_t nx = g.nx(), n = g.num_nodes();
    if (A.rows() != n || A.cols() != n) throw std::invalid_argument("csr_to_9: size mismatch");
    std::memset(coef, 0, sizeof(double) * 9 * static_cast<std::size_t>(n));
    for (std::int32_t i = 0; i < n; ++i) {
        const std::int32_t gx = i % nx, gy = i / nx;
        for (std::int32_t k = A.row_ptr()[i]; k < A.row_ptr()[i + 1]; ++k) {
            const std::int32_t j = A.col_idx()[k];
            const std::int32_t dx = j % nx - gx, dy = j / nx - gy;
            if (dx < -1 || dx > 1 || dy < -1 || dy > 1)
                throw std::runtime_error("csr_to_9: entry outside the 9-point stencil");
            coef[static_cast<std::size_t>((dy + 1) * 3 + (dx + 1)) * n + i] = A.values()[k];
        }
    }
}

SparseMatrix nine_to_csr(const double* coef, int level)
{
    const Grid g(level);
    const std::int32_t nx = g.nx(), n = g.num_nodes();
    std::vector<Triplet> t;
    t.reserve(static_cast<std::size_t>(n) * 9);
    for (std::int32_t i = 0; i < n; ++i) {
        const std::int32_t gx = i % nx, gy = i / nx;
        for (int d = 0; d < 9; ++d) {
            const int dx = d % 3 - 1, dy = d / 3 - 1;
            const std::int32_t jx = gx + dx, jy = gy + dy;
            if (jx < 0 || jx >= nx || jy < 0 || jy >= nx) continue;
            t.push_back({i, jy * nx + jx, coef[static_cast<std::size_t>(d) * n + i]});
        }
    }
    return SparseMatrix::from_triplets(n, n, std::move(t));
}

struct Handle {
    ControlProblem problem;
    std::unique_ptr<Grid> grid;
    bool heat = false;
    std::unique_ptr<QpProblem> qp;
    std::unique_ptr<SpaceTimeSystem> sys;
    IpmModel model;
    std::size_t ny = 0, nu = 0;

    // preconditioners from the last ref_precond_setup
    ThetaBlocks theta;
    std::optional<BlockDiagPrecond> pd;
    std::optional<BlockTriPrecond> pt;
    std::optional<PermutedPrecond> ppi;
    std::optional<SchurApprox> schur;
    // heat compositions (timedep.cpp:373-426)
    std::vector<ChebyshevSemiIteration> heat_cheb;
    Vector ad, bd, cd;
    std::optional<TimeSchurApprox> heat_schur;
    // bounded Krylov sample (bench.py reference arm): first Newton system
    Vector sample_rhs;
    bool sample_ready = false;
};

struct CapturedNewton {}; // aborts ipm_solve after the first Newton system is formed

MgOptions mg_options(const Handle& h, const ref_params& p)
{
    MgOptions mg;
    mg.level = h.grid->level;
    mg.cycles = p.mg_cycles;
    mg.pre = p.mg_pre;
    mg.post = p.mg_post;
    if (!h.heat) mg.rediscretize = h.qp->op_assembler;
    return mg;
}

IpmParams to_params(const ref_params& p)
{
    IpmParams q;
    q.alpha0 = p.alpha0;
    q.sigma = p.sigma;
    q.eps_p = p.eps_p;
    q.eps_d = p.eps_d;
    q.eps_c = p.eps_c;
    q.mu0 = p.mu0;
    q.max_iterations = p.max_iterations;
    q.linear_tol = p.linear_tol;
    q.linear_maxit = p.linear_maxit;
    q.cheb_steps = p.cheb_steps;
    q.mg_cycles = p.mg_cycles;
    q.mg_pre = p.mg_pre;
    q.mg_post = p.mg_post;
    switch (p.solver) {
    case 0: q.solver = SolverKind::gmres_pt; break;
    case 1: q.solver = SolverKind::minres_pd; break;
    case 2: q.solver = SolverKind::gmres_ppi; break;
    case 3: q.solver = SolverKind::dense; break;
    case 10: q.solver = SolverKind::gmres_pt; break; // overridden below
    default: throw std::invalid_argument("ref: unknown solver code");
    }
    return q;
}

// Heat block preconditioner pieces exactly as timedep.cpp:373-395 builds them.
void heat_setup(Handle& h, const ThetaBlocks& theta, const ref_params& p)
{
    const SpaceTimeSystem& s = *h.sys;
    const std::size_t nn = static_cast<std::size_t>(s.n);
    const std::size_t ny = nn * static_cast<std::size_t>(s.nt);
    h.heat_cheb.clear();
    h.heat_cheb.reserve(static_cast<std::size_t>(s.nt));
    for (int k = 0; k < s.nt; ++k) {
        Vector th(theta.theta_y.begin() + static_cast<std::ptrdiff_t>(k * nn),
                  theta.theta_y.begin() + static_cast<std::ptrdiff_t>((k + 1) * nn));
        h.heat_cheb.emplace_back(s.M, s.tau * s.qweights[static_cast<std::size_t>(k)],
                                 std::move(th), p.cheb_steps);
    }
    const Vector dM = s.M.diagonal_vector();
    h.ad.resize(ny);
    h.bd.resize(ny);
    h.cd.resize(ny);
    for (int k = 0; k < s.nt; ++k) {
        const double sc = s.alpha * s.tau * s.qweights[static_cast<std::size_t>(k)];
        const std::size_t off = static_cast<std::size_t>(k) * nn;
        for (std::size_t i = 0; i < nn; ++i) {
            h.ad[off + i] = sc * dM[i] + theta.theta_w[off + i];
            h.bd[off + i] = -sc * dM[i];
            h.cd[off + i] = sc * dM[i] + theta.theta_v[off + i];
        }
    }
    MgOptions mg = mg_options(h, p);
    h.heat_schur.emplace(s, theta, InnerSolve::multigrid, mg);
}

// timedep.cpp:396-426 (block_triangular = true) and its block-diagonal
// counterpart (no coupling row) used by the harness MINRES composition.
Vector heat_apply(const Handle& h, const Vector& r, bool triangular)
{
    const SpaceTimeSystem& s = *h.sys;
    const std::size_t nn = static_cast<std::size_t>(s.n);
    const std::size_t ny = nn * static_cast<std::size_t>(s.nt);
    Vector ry(r.begin(), r.begin() + static_cast<std::ptrdiff_t>(ny));
    Vector rw(r.begin() + static_cast<std::ptrdiff_t>(ny), r.begin() + static_cast<std::ptrdiff_t>(2 * ny));
    Vector rv(r.begin() + static_cast<std::ptrdiff_t>(2 * ny), r.begin() + static_cast<std::ptrdiff_t>(3 * ny));
    Vector rp(r.begin() + static_cast<std::ptrdiff_t>(3 * ny), r.end());
    Vector vy(ny);
    for (int k = 0; k < s.nt; ++k) {
        const std::size_t off = static_cast<std::size_t>(k) * nn;
        Vector slice(ry.begin() + static_cast<std::ptrdiff_t>(off),
                     ry.begin() + static_cast<std::ptrdiff_t>(off + nn));
        const Vector sol = h.heat_cheb[static_cast<std::size_t>(k)].apply(slice);
        std::copy(sol.begin(), sol.end(), vy.begin() + static_cast<std::ptrdiff_t>(off));
    }
    Vector vw, vv;
    block_2x2_inverse_apply(h.ad, h.bd, h.bd, h.cd, rw, rv, vw, vv);
    Vector vp;
    if (triangular) {
        Vector t = s.apply_bidiag(vy);
        Vector zc(2 * ny);
        std::copy(vw.begin(), vw.end(), zc.begin());
        std::copy(vv.begin(), vv.end(), zc.begin() + static_cast<std::ptrdiff_t>(ny));
        const Vector cz = s.apply_coupling(zc);
        for (std::size_t i = 0; i < ny; ++i) t[i] += -cz[i] - rp[i];
        vp = h.heat_schur->apply_inverse(t);
    } else {
        vp = h.heat_schur->apply_inverse(rp);
    }
    Vector out(r.size());
    std::copy(vy.begin(), vy.end(), out.begin());
    std::copy(vw.begin(), vw.end(), out.begin() + static_cast<std::ptrdiff_t>(ny));
    std::copy(vv.begin(), vv.end(), out.begin() + static_cast<std::ptrdiff_t>(2 * ny));
    std::copy(vp.begin(), vp.end(), out.begin() + static_cast<std::ptrdiff_t>(3 * ny));
    return out;
}

// BASELINE config 5 asks for MINRES on the heat problem; the reference heat
// path is gmres-pt only (timedep.cpp:429-431), so this composes reference
// classes (per-block Chebyshev, block_2x2_inverse_apply, TimeSchurApprox,
// minres) into a block-diagonal MINRES newton_solve.
void install_heat_minres(Handle& h)
{
    Handle* hp = &h;
    h.model.newton_solve = [hp](const ThetaBlocks& theta, const Vector& r1, const Vector& r2,
                                const Vector& r3, const IpmParams& params) {
        Handle& hh = *hp;
        ref_params rp{};
        rp.cheb_steps = params.cheb_steps;
        rp.mg_cycles = params.mg_cycles;
        rp.mg_pre = params.mg_pre;
        rp.mg_post = params.mg_post;
        heat_setup(hh, theta, rp);
        IpmModel mv = make_spacetime_model(*hh.sys);
        const LinearOperator A = make_saddle_operator(mv, theta);
        const Vector rhs = concat(concat(r1, r2), r3);
        const LinearOperator P{A.n, [&hh](const Vector& r, Vector& out) {
                                   out = heat_apply(hh, r, false);
                               }};
        Vector x;
        SolveReport rep = minres(A, P, rhs, x, params.linear_tol, params.linear_maxit);
        const std::size_t ny = hh.ny;
        NewtonSolveResult out;
        out.dy.assign(x.begin(), x.begin() + static_cast<std::ptrdiff_t>(ny));
        out.dz.assign(x.begin() + static_cast<std::ptrdiff_t>(ny), x.begin() + static_cast<std::ptrdiff_t>(3 * ny));
        out.dp.assign(x.begin() + static_cast<std::ptrdiff_t>(3 * ny), x.end());
        out.report = std::move(rep);
        return out;
    };
}

double model_objective(const Handle& h, const Vector& y, const Vector& z)
{
    if (!h.heat) return h.qp->objective(y, z);
    // J = 1/2 (y-y_d)' hy (y-y_d) + 1/2 z' hz z + beta_grad' z
    Vector diff = y;
    axpy(-1.0, h.model.y_d, diff);
    double val = 0.5 * dot(diff, h.model.hy(diff));
    val += 0.5 * dot(z, h.model.hz(z));
    val += dot(h.model.beta_grad, z);
    return val;
}

} // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

void* ref_problem_create(const ref_problem_desc* d)
{
    Handle* out = nullptr;
    const int rc = guarded([&] {
        auto h = std::make_unique<Handle>();
        h->grid = std::make_unique<Grid>(d->level);
        const std::size_t n = static_cast<std::size_t>(h->grid->num_nodes());
        ControlProblem& p = h->problem;
        p.pde = d->pde == 0 ? PdeKind::poisson : d->pde == 1 ? PdeKind::convdiff : PdeKind::heat;
        p.eps = d->eps;
        p.tau = d->tau;
        p.horizon = d->horizon;
        p.alpha = d->alpha;
        p.beta = d->beta;
        p.y_d = from_ptr(d->y_d, n); // heat: first slice; replaced below
        p.f = d->f ? from_ptr(d->f, n) : Vector(n, 0.0);
        p.u_a = from_ptr(d->u_a, n);
        p.u_b = from_ptr(d->u_b, n);
        if (d->y_a) {
            p.y_a = from_ptr(d->y_a, n);
            p.y_b = from_ptr(d->y_b, n);
        }
        if (d->has_obs) p.observation = ObservationRegion{d->obs[0], d->obs[1], d->obs[2], d->obs[3]};
        if (p.pde == PdeKind::heat) {
            h->heat = true;
            h->sys = std::make_unique<SpaceTimeSystem>(assemble_spacetime(
                p, *h->grid, d->quadrature ? TimeQuadrature::trapezoid : TimeQuadrature::rectangle));
            const std::size_t ny = n * static_cast<std::size_t>(h->sys->nt);
            if (static_cast<std::size_t>(d->y_d_len) == ny)
                h->sys->y_d = from_ptr(d->y_d, ny); // public field, copied by the model
            else if (static_cast<std::size_t>(d->y_d_len) != n)
                throw std::invalid_argument("ref: heat y_d must have n or n*nt entries");
            h->model = make_spacetime_model(*h->sys);
            h->ny = h->nu = ny;
        } else {
            if (static_cast<std::size_t>(d->y_d_len) != n)
                throw std::invalid_argument("ref: y_d must have n entries");
            h->qp = std::make_unique<QpProblem>(build_qp(p, *h->grid));
            h->model = make_steady_model(*h->qp);
            h->ny = h->nu = n;
        }
        out = h.release();
    });
    return rc == 0 ? out : nullptr;
}

void ref_problem_destroy(void* h) { delete static_cast<Handle*>(h); }

int ref_problem_sizes(void* hv, int* n, int* nt, int* has_sb)
{
    return guarded([&] {
        Handle& h = *static_cast<Handle*>(hv);
        *n = h.grid->num_nodes();
        *nt = h.heat ? h.sys->nt : 1;
        *has_sb = h.model.has_state_bounds() ? 1 : 0;
    });
}

int ref_ipm_solve(void* hv, const ref_params* pp, ref_result* r)
{
    return guarded([&] {
        Handle& h = *static_cast<Handle*>(hv);
        IpmParams params = to_params(*pp);
        const auto saved = h.model.newton_solve;
        if (pp->solver == 10) {
            if (!h.heat) throw std::invalid_argument("ref: solver 10 is the heat MINRES composition");
            install_heat_minres(h);
        }
        double newton_total = 0.0;
        std::vector<double> newton_each;
        IpmModel model = h.model;
        const auto inner = model.newton_solve;
        model.newton_solve = [&](const ThetaBlocks& th, const Vector& a, const Vector& b,
                                 const Vector& c, const IpmParams& prm) {
            const double t0 = now_s();
            NewtonSolveResult res = inner(th, a, b, c, prm);
            const double dt = now_s() - t0;
            newton_total += dt;
            newton_each.push_back(dt);
            return res;
        };
        const double t0 = now_s();
        IpmResult res;
        try {
            res = ipm_solve(model, params);
        } catch (...) {
            h.model.newton_solve = saved;
            throw;
        }
        r->solve_seconds = now_s() - t0;
        h.model.newton_solve = saved;
        r->newton_seconds = newton_total;

        const auto& st = res.state;
        to_ptr(st.y, r->y);
        to_ptr(st.z, r->z);
        to_ptr(st.p, r->p);
        if (h.model.has_state_bounds()) {
            to_ptr(st.lam_ya, r->lam_ya);
            to_ptr(st.lam_yb, r->lam_yb);
        }
        to_ptr(st.lam_za, r->lam_za);
        to_ptr(st.lam_zb, r->lam_zb);
        to_ptr(res.u, r->u);
        r->n_records = static_cast<int>(res.stats.iterations.size());
        long long tot = 0;
        for (std::size_t k = 0; k < res.stats.iterations.size(); ++k) {
            const auto& it = res.stats.iterations[k];
            tot += it.lin_iters;
            if (r->records && static_cast<int>(k) < r->records_cap) {
                ref_record& rec = r->records[k];
                rec.k = it.k;
                rec.mu = it.mu;
                rec.norm_xp = it.norm_xp;
                rec.norm_xd = it.norm_xd;
                rec.norm_xc = it.norm_xc;
                rec.lin_iters = it.lin_iters;
                rec.lin_relres = it.lin_relres;
                rec.lin_converged = it.lin_converged ? 1 : 0;
                rec.newton_seconds = (k >= 1 && k - 1 < newton_each.size()) ? newton_each[k - 1] : 0.0;
            }
        }
        r->total_lin = tot;
        r->nli = res.stats.nli;
        r->converged = res.stats.converged ? 1 : 0;
        r->av_li = res.stats.av_li;
        r->mu = st.mu;
        r->objective = model_objective(h, st.y, st.z);
        r->sparsity_pct = res.sparsity.percent_below_threshold;
        r->l1 = res.sparsity.l1_norm;
        // nodal sparsity over the closed grid (bench.cpp:85-99)
        const std::int64_t nx = h.grid->nx();
        const std::int64_t all = (nx + 2) * (nx + 2);
        const std::int64_t nt = h.heat ? h.sys->nt : 1;
        std::int64_t below = 0;
        for (double v : res.u)
            if (std::abs(v) < 1e-2) ++below;
        below += (all - nx * nx) * nt;
        r->nodal_sparsity_pct = 100.0 * static_cast<double>(below) / static_cast<double>(all * nt);
    });
}

int ref_kkt_apply(void* hv, const double* ty, const double* tw, const double* tv, const double* x,
                  double* out)
{
    return guarded([&] {
        Handle& h = *static_cast<Handle*>(hv);
        ThetaBlocks th{from_ptr(ty, h.ny), from_ptr(tw, h.nu), from_ptr(tv, h.nu)};
        const LinearOperator A = make_saddle_operator(h.model, th);
        Vector o(static_cast<std::size_t>(A.n));
        A.apply_fn(from_ptr(x, static_cast<std::size_t>(A.n)), o);
        to_ptr(o, out);
    });
}

int ref_precond_setup(void* hv, const double* ty, const double* tw, const double* tv,
                      const ref_params* pp)
{
    return guarded([&] {
        Handle& h = *static_cast<Handle*>(hv);
        h.theta = ThetaBlocks{from_ptr(ty, h.ny), from_ptr(tw, h.nu), from_ptr(tv, h.nu)};
        h.pd.reset();
        h.pt.reset();
        h.ppi.reset();
        h.schur.reset();
        if (h.heat) {
            heat_setup(h, h.theta, *pp);
            return;
        }
        const QpProblem& q = *h.qp;
        const MgOptions mg = mg_options(h, *pp);
        const ThetaBlocks& th = h.theta;
        if (q.partial_observation) {
            h.ppi.emplace(q.L, q.M_obs, q.M, q.alpha, th, InnerSolve::multigrid, mg);
            return;
        }
        auto make_b11 = [&] {
            return Block11Approx(q.M_obs, th.theta_y, q.M, q.alpha, th.theta_w, th.theta_v,
                                 InnerSolve::multigrid, pp->cheb_steps);
        };
        auto make_schur = [&] {
            return SchurApprox(q.L, q.M_obs, th.theta_y,
                               build_m_hat(q.alpha, q.M.diagonal_vector(), th.theta_w,
                                           th.theta_v, th.theta_y),
                               InnerSolve::multigrid, mg);
        };
        h.pd.emplace(make_b11(), make_schur());
        h.pt.emplace(make_b11(), make_schur(), q.L, q.M);
        h.schur.emplace(make_schur());
    });
}

int ref_precond_apply(void* hv, int kind, const double* r, double* out)
{
    return guarded([&] {
        Handle& h = *static_cast<Handle*>(hv);
        const Vector rv = from_ptr(r, 2 * h.ny + 2 * h.nu);
        Vector o;
        switch (kind) {
        case 0: if (!h.pd) throw std::invalid_argument("ref: P_D not set up"); o = h.pd->apply(rv); break;
        case 1: if (!h.pt) throw std::invalid_argument("ref: P_T not set up"); o = h.pt->apply(rv); break;
        case 2: if (!h.ppi) throw std::invalid_argument("ref: P_Pi not set up"); o = h.ppi->apply(rv); break;
        case 3: if (!h.heat_schur) throw std::invalid_argument("ref: heat not set up"); o = heat_apply(h, rv, true); break;
        case 4: if (!h.heat_schur) throw std::invalid_argument("ref: heat not set up"); o = heat_apply(h, rv, false); break;
        default: throw std::invalid_argument("ref: unknown preconditioner kind");
        }
        to_ptr(o, out);
    });
}

int ref_schur_apply(void* hv, const double* r, double* out)
{
    return guarded([&] {
        Handle& h = *static_cast<Handle*>(hv);
        if (h.heat) {
            if (!h.heat_schur) throw std::invalid_argument("ref: heat not set up");
            to_ptr(h.heat_schur->apply_inverse(from_ptr(r, h.ny)), out);
            return;
        }
        if (!h.schur) throw std::invalid_argument("ref: Schur approximation not set up");
        to_ptr(h.schur->apply_inverse(from_ptr(r, h.ny)), out);
    });
}

int ref_time_applies(void* hv, int kind, int reps, const double* x, double* kkt_s, double* prec_s)
{
    return guarded([&] {
        Handle& h = *static_cast<Handle*>(hv);
        const LinearOperator A = make_saddle_operator(h.model, h.theta);
        const Vector xv = from_ptr(x, static_cast<std::size_t>(A.n));
        Vector o(xv.size());
        double t0 = now_s();
        for (int i = 0; i < reps; ++i) A.apply_fn(xv, o);
        *kkt_s = (now_s() - t0) / reps;
        std::vector<double> tmp(xv.size());
        t0 = now_s();
        for (int i = 0; i < reps; ++i) {
            if (ref_precond_apply(hv, kind, xv.data(), tmp.data()) != 0)
                throw std::runtime_error(g_err);
        }
        *prec_s = (now_s() - t0) / reps;
    });
}

int ref_newton_sample_prepare(void* hv, const ref_params* pp, double* setup_s)
{
    return guarded([&] {
        Handle& h = *static_cast<Handle*>(hv);
        IpmParams params = to_params(*pp);
        IpmModel model = h.model;
        ThetaBlocks theta;
        Vector r1, r2, r3;
        // the reference's own ipm_solve forms the first Newton system (initial
        // point, mu <- sigma mu0, build_theta, newton_rhs: ipm.cpp:278-300)
        model.newton_solve = [&](const ThetaBlocks& th, const Vector& a, const Vector& b,
                                 const Vector& c, const IpmParams&) -> NewtonSolveResult {
            theta = th;
            r1 = a;
            r2 = b;
            r3 = c;
            throw CapturedNewton{};
        };
        try {
            (void)ipm_solve(model, params);
            throw std::runtime_error("ref: ipm_solve converged before a Newton step");
        } catch (const CapturedNewton&) {
        }
        if (theta.theta_y.empty()) theta.theta_y.assign(h.ny, 0.0);
        const double t0 = now_s();
        if (ref_precond_setup(hv, theta.theta_y.data(), theta.theta_w.data(),
                              theta.theta_v.data(), pp) != 0)
            throw std::runtime_error(g_err);
        *setup_s = now_s() - t0;
        h.theta = theta;
        h.sample_rhs = concat(concat(r1, r2), r3);
        h.sample_ready = true;
    });
}

int ref_newton_sample_run(void* hv, int kind, int method, double tol, int maxit, int* iters,
                          double* relres, double* seconds)
{
    return guarded([&] {
        Handle& h = *static_cast<Handle*>(hv);
        if (!h.sample_ready) throw std::invalid_argument("ref: newton sample not prepared");
        const LinearOperator A = make_saddle_operator(h.model, h.theta);
        const LinearOperator P{A.n, [&h, kind](const Vector& r, Vector& out) {
                                   out.resize(r.size());
                                   if (ref_precond_apply(&h, kind, r.data(), out.data()) != 0)
                                       throw std::runtime_error(g_err);
                               }};
        Vector x;
        const double t0 = now_s();
        SolveReport rep = method == 0 ? gmres(A, P, h.sample_rhs, x, tol, maxit)
                                      : minres(A, P, h.sample_rhs, x, tol, maxit);
        *seconds = now_s() - t0;
        *iters = rep.iterations;
        *relres = rep.relative_residual;
    });
}

int ref_objective(void* hv, const double* y, const double* z, double* out)
{
    return guarded([&] {
        Handle& h = *static_cast<Handle*>(hv);
        *out = model_objective(h, from_ptr(y, h.ny), from_ptr(z, 2 * h.nu));
    });
}

int ref_ipm_pieces(void* hv, const double* y, const double* z, const double* p,
                   const double* lam_ya, const double* lam_yb, const double* lam_za,
                   const double* lam_zb, double mu_state, double mu_rhs, double* theta_y,
                   double* theta_w, double* theta_v, double* r1, double* r2, double* r3,
                   double* norms3)
{
    return guarded([&] {
        Handle& h = *static_cast<Handle*>(hv);
        IpmState s;
        s.y = from_ptr(y, h.ny);
        s.z = from_ptr(z, 2 * h.nu);
        s.p = from_ptr(p, h.ny);
        if (h.model.has_state_bounds()) {
            s.lam_ya = from_ptr(lam_ya, h.ny);
            s.lam_yb = from_ptr(lam_yb, h.ny);
        }
        s.lam_za = from_ptr(lam_za, 2 * h.nu);
        s.lam_zb = from_ptr(lam_zb, 2 * h.nu);
        s.mu = mu_state;
        const ThetaBlocks th = build_theta(h.model, s);
        to_ptr(th.theta_y, theta_y);
        to_ptr(th.theta_w, theta_w);
        to_ptr(th.theta_v, theta_v);
        Vector a, b, c;
        newton_rhs(h.model, s, mu_rhs, a, b, c);
        to_ptr(a, r1);
        to_ptr(b, r2);
        to_ptr(c, r3);
        const IpmResiduals res = ipm_residuals(h.model, s);
        norms3[0] = res.norm_xp;
        norms3[1] = res.norm_xd;
        norms3[2] = res.norm_xc;
    });
}

int ref_assemble9(int what, int level, double eps, const double* obs, double* coef)
{
    return guarded([&] {
        const Grid g(level);
        SparseMatrix A;
        switch (what) {
        case 0: A = assemble_mass(g, MassVariant::consistent); break;
        case 1: A = assemble_stiffness_poisson(g); break;
        case 2: A = assemble_convdiff(g, eps, default_wind(), true); break;
        case 3: A = assemble_partial_mass(g, ObservationRegion{obs[0], obs[1], obs[2], obs[3]}); break;
        case 4: {
            const Vector d = assemble_mass(g, MassVariant::consistent).row_sums();
            to_ptr(d, coef);
            return;
        }
        default: throw std::invalid_argument("ref_assemble9: unknown operator");
        }
        csr_to_9(A, level, coef);
    });
}

struct MgHandle {
    int level;
    MgHierarchy h;
};

void* ref_mg_create(int level, const double* coef9, int redisc, double eps, int transpose_base)
{
    MgHandle* out = nullptr;
    guarded([&] {
        MgOptions o;
        o.level = level;
        if (redisc) {
            if (transpose_base)
                o.rediscretize = [eps](int l) {
                    return assemble_convdiff(Grid(l), eps, default_wind(), true).transposed();
                };
            else
                o.rediscretize = [eps](int l) {
                    return assemble_convdiff(Grid(l), eps, default_wind(), true);
                };
        }
        out = new MgHandle{level, MgHierarchy::build(nine_to_csr(coef9, level), o)};
    });
    return out;
}

int ref_mg_solve(void* mv, const double* rhs, int cycles, int pre, int post, double* out)
{
    return guarded([&] {
        MgHandle& m = *static_cast<MgHandle*>(mv);
        const std::size_t n = static_cast<std::size_t>(Grid(m.level).num_nodes());
        to_ptr(m.h.solve(from_ptr(rhs, n), cycles, pre, post), out);
    });
}

int ref_mg_depth(void* mv) { return static_cast<MgHandle*>(mv)->h.depth(); }

int ref_mg_level_matrix(void* mv, int k, double* coef9)
{
    return guarded([&] {
        MgHandle& m = *static_cast<MgHandle*>(mv);
        csr_to_9(m.h.level_matrix(static_cast<std::size_t>(k)), m.level - k, coef9);
    });
}

void ref_mg_destroy(void* mv) { delete static_cast<MgHandle*>(mv); }

int ref_gs_sweep(int level, const double* coef9, const double* b, double* x, int forward)
{
    return guarded([&] {
        const SparseMatrix A = nine_to_csr(coef9, level);
        const std::size_t n = static_cast<std::size_t>(A.rows());
        Vector xv = from_ptr(x, n);
        gauss_seidel_sweep(A, from_ptr(b, n), xv, forward != 0);
        to_ptr(xv, x);
    });
}

int ref_cheb_apply(int level, double scale, const double* extra, int steps, const double* b,
                   double* x)
{
    return guarded([&] {
        const Grid g(level);
        const std::size_t n = static_cast<std::size_t>(g.num_nodes());
        const SparseMatrix M = assemble_mass(g, MassVariant::consistent);
        ChebyshevSemiIteration c(M, scale, extra ? from_ptr(extra, n) : Vector(n, 0.0), steps);
        to_ptr(c.apply(from_ptr(b, n)), x);
    });
}

int ref_krylov_9diag(int method, int level, const double* coef9, const double* b, double tol,
                     int maxit, double* x, int* iters, double* relres)
{
    return guarded([&] {
        const SparseMatrix A = nine_to_csr(coef9, level);
        const std::size_t n = static_cast<std::size_t>(A.rows());
        const Vector d = A.diagonal_vector();
        const LinearOperator op = LinearOperator::from_matrix(A);
        const LinearOperator P{A.rows(), [&d](const Vector& r, Vector& o) {
                                   o.resize(r.size());
                                   for (std::size_t i = 0; i < r.size(); ++i) o[i] = r[i] / d[i];
                               }};
        Vector xv;
        SolveReport rep = method == 0 ? minres(op, P, from_ptr(b, n), xv, tol, maxit)
                                      : gmres(op, P, from_ptr(b, n), xv, tol, maxit);
        to_ptr(xv, x);
        *iters = rep.iterations;
        *relres = rep.relative_residual;
    });
}

} // extern "C"
