// C++ façade over the optcon-b200 C ABI that mirrors the reference solver API
// (/root/reference/proj/include/optcon/{qp,ipm,krylov,timedep}.hpp), so a caller
// of the reference switches by changing the include and the namespace:
//
//     optcon::QpProblem qp = optcon::build_qp(problem, grid);            // reference
//     optcon::IpmResult r  = optcon::ipm_solve(optcon::make_steady_model(qp), params);
//
//     optcon_b200::QpProblem qp = optcon_b200::build_qp(problem, grid);   // B200
//     optcon_b200::IpmResult r  = optcon_b200::ipm_solve(qp, params);
//
// Value-semantic std::vector<double> in and out, std::invalid_argument /
// std::runtime_error with the reference's messages, one Context (CUDA stream)
// per host thread. Header-only; link with -loptcon_b200.
#pragma once

#include "optcon_b200.h"

#include <cmath>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

namespace optcon_b200 {

using Vector = std::vector<double>;

inline void check(int rc)
{
    if (rc == OC_OK) return;
    const std::string msg = oc_last_error();
    if (rc == OC_INVALID_ARGUMENT) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}

enum class PdeKind { poisson = OC_PDE_POISSON, convdiff = OC_PDE_CONVDIFF, heat = OC_PDE_HEAT };
enum class SolverKind { gmres_pt = OC_SOLVER_GMRES_PT, minres_pd = OC_SOLVER_MINRES_PD,
                        gmres_ppi = OC_SOLVER_GMRES_PPI };

/// grid.hpp:14-37
struct Grid {
    int level;
    explicit Grid(int l) : level(l)
    {
        if (level < 1 || level > 14) throw std::invalid_argument("Grid: level out of range");
    }
    double h() const { return 1.0 / double(1 << level); }
    int nx() const { return (1 << level) - 1; }
    int num_nodes() const { return nx() * nx(); }
};

struct ObservationRegion {
    double a1, b1, a2, b2;
};

/// qp.hpp:20-34
struct ControlProblem {
    PdeKind pde = PdeKind::poisson;
    double eps = 1e-1, tau = 0.04, horizon = 1.0;
    double alpha = 1e-2, beta = 1e-2;
    Vector y_d, f, u_a, u_b;
    std::optional<Vector> y_a, y_b;
    std::optional<ObservationRegion> observation;
};

/// ipm.hpp:17-32
struct IpmParams {
    double alpha0 = 0.995, sigma = 0.2, eps_p = 1e-6, eps_d = 1e-6, eps_c = 1e-6, mu0 = 1.0;
    int max_iterations = 100;
    double linear_tol = 1e-10;
    int linear_maxit = 200, cheb_steps = 20, mg_cycles = 3, mg_pre = 5, mg_post = 5;
    SolverKind solver = SolverKind::gmres_pt;
    int gmres_restart = 0;
    /// OC_SMOOTHER_COLOR4 (parallel default) or OC_SMOOTHER_LEX (the
    /// reference's lexicographic Gauss-Seidel, faithful mode)
    int smoother = OC_SMOOTHER_AUTO;

    oc_ipm_params c() const
    {
        oc_ipm_params p{};
        p.alpha0 = alpha0; p.sigma = sigma; p.eps_p = eps_p; p.eps_d = eps_d; p.eps_c = eps_c;
        p.mu0 = mu0; p.max_iterations = max_iterations; p.linear_tol = linear_tol;
        p.linear_maxit = linear_maxit; p.cheb_steps = cheb_steps; p.mg_cycles = mg_cycles;
        p.mg_pre = mg_pre; p.mg_post = mg_post; p.solver = static_cast<int>(solver);
        p.smoother = smoother; p.gmres_restart = gmres_restart;
        return p;
    }
};

/// ipm.hpp:36-60, 100-105
struct IpmState {
    Vector y, z, p, lam_ya, lam_yb, lam_za, lam_zb;
    double mu = 1.0;
    int k = 0;
};
struct IterationRecord {
    int k = 0;
    double mu = 0, norm_xp = 0, norm_xd = 0, norm_xc = 0;
    int lin_iters = 0;
    double lin_relres = 0;
    bool lin_converged = true;
};
struct IpmStats {
    std::vector<IterationRecord> iterations;
    bool converged = false;
    int nli = 0;
    double av_li = 0.0;
};
struct SparsityReport {
    double percent_below_threshold, l1_norm;
};
struct IpmResult {
    IpmState state;
    Vector u;
    SparsityReport sparsity{0, 0};
    IpmStats stats;
    double objective = 0.0;
};

/// One device context (CUDA stream) per host thread.
class Context {
public:
    explicit Context(int device = 0) { check(oc_create(&h_, device)); }
    ~Context() { oc_destroy(h_); }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;
    oc_ctx* get() const { return h_; }

private:
    oc_ctx* h_ = nullptr;
};

inline Context& default_context()
{
    thread_local Context ctx(0);
    return ctx;
}

/// Device-resident QpProblem / SpaceTimeSystem (qp.hpp:53-77, timedep.hpp:13-40).
class QpProblem {
public:
    QpProblem(const ControlProblem& p, const Grid& g, Context& ctx = default_context())
    {
        oc_problem_desc d{};
        d.pde = static_cast<int>(p.pde);
        d.level = g.level;
        d.eps = p.eps;
        d.tau = p.tau;
        d.horizon = p.horizon;
        d.alpha = p.alpha;
        d.beta = p.beta;
        d.y_d = p.y_d.data();
        d.y_d_len = static_cast<long long>(p.y_d.size());
        const size_t n = static_cast<size_t>(g.num_nodes());
        if (p.u_a.size() != n || p.u_b.size() != n || (!p.f.empty() && p.f.size() != n))
            throw std::invalid_argument("build_qp: nodal data size mismatch with grid");
        d.f = p.f.empty() ? nullptr : p.f.data();
        d.u_a = p.u_a.data();
        d.u_b = p.u_b.data();
        if (p.y_a.has_value() != p.y_b.has_value())
            throw std::invalid_argument("ControlProblem: state bounds must come as a pair");
        d.y_a = p.y_a ? p.y_a->data() : nullptr;
        d.y_b = p.y_b ? p.y_b->data() : nullptr;
        if (p.observation) {
            d.has_obs = 1;
            d.obs[0] = p.observation->a1; d.obs[1] = p.observation->b1;
            d.obs[2] = p.observation->a2; d.obs[3] = p.observation->b2;
        }
        oc_problem* h = nullptr;
        check(oc_problem_create(ctx.get(), &d, &h));
        h_.reset(h);
        check(oc_problem_info_get(h, &info_));
    }
    oc_problem* get() const { return h_.get(); }
    const oc_problem_info& info() const { return info_; }

private:
    struct Del {
        void operator()(oc_problem* p) const { oc_problem_destroy(p); }
    };
    std::unique_ptr<oc_problem, Del> h_;
    oc_problem_info info_{};
};

/// qp.hpp:82 (steady) — heat goes through assemble_spacetime.
inline QpProblem build_qp(const ControlProblem& p, const Grid& g, Context& ctx = default_context())
{
    if (p.pde == PdeKind::heat)
        throw std::invalid_argument("build_qp: heat problems use the space-time assembly");
    return QpProblem(p, g, ctx);
}

/// timedep.hpp:68
inline QpProblem assemble_spacetime(const ControlProblem& p, const Grid& g,
                                    Context& ctx = default_context())
{
    if (p.pde != PdeKind::heat)
        throw std::invalid_argument("assemble_spacetime: expects the heat problem");
    return QpProblem(p, g, ctx);
}

/// ipm.hpp:134 — the whole interior-point loop on the device.
inline IpmResult ipm_solve(const QpProblem& qp, const IpmParams& params = IpmParams{})
{
    const size_t ny = static_cast<size_t>(qp.info().ny);
    IpmResult r;
    r.state.y.resize(ny);
    r.state.z.resize(2 * ny);
    r.state.p.resize(ny);
    r.state.lam_za.resize(2 * ny);
    r.state.lam_zb.resize(2 * ny);
    if (qp.info().has_state_bounds) {
        r.state.lam_ya.resize(ny);
        r.state.lam_yb.resize(ny);
    }
    r.u.resize(ny);
    std::vector<oc_iter_record> recs(static_cast<size_t>(params.max_iterations) + 1);
    oc_ipm_result out{};
    out.y = r.state.y.data();
    out.z = r.state.z.data();
    out.p = r.state.p.data();
    out.lam_ya = r.state.lam_ya.empty() ? nullptr : r.state.lam_ya.data();
    out.lam_yb = r.state.lam_yb.empty() ? nullptr : r.state.lam_yb.data();
    out.lam_za = r.state.lam_za.data();
    out.lam_zb = r.state.lam_zb.data();
    out.u = r.u.data();
    out.records = recs.data();
    out.records_cap = static_cast<int>(recs.size());
    const oc_ipm_params p = params.c();
    check(oc_ipm_solve(qp.get(), &p, &out));
    for (int i = 0; i < out.n_records && i < out.records_cap; ++i) {
        const oc_iter_record& a = recs[static_cast<size_t>(i)];
        r.stats.iterations.push_back({a.k, a.mu, a.norm_xp, a.norm_xd, a.norm_xc, a.lin_iters,
                                      a.lin_relres, a.lin_converged != 0});
    }
    r.stats.converged = out.converged != 0;
    r.stats.nli = out.nli;
    r.stats.av_li = out.av_li;
    r.state.mu = out.mu;
    r.state.k = out.nli;
    r.sparsity = {out.sparsity_pct, out.l1};
    r.objective = out.objective;
    return r;
}

/// timedep.hpp:88-91
inline IpmResult solve_heat_control(const ControlProblem& p, const Grid& g,
                                    const IpmParams& params = IpmParams{},
                                    Context& ctx = default_context())
{
    return ipm_solve(assemble_spacetime(p, g, ctx), params);
}

/// ThetaBlocks (precond.hpp:16-20) + make_saddle_operator(model, theta).apply
inline Vector saddle_apply(const QpProblem& qp, const Vector& theta_y, const Vector& theta_w,
                           const Vector& theta_v, const Vector& x)
{
    Vector out(x.size());
    check(oc_kkt_apply(qp.get(), theta_y.empty() ? nullptr : theta_y.data(), theta_w.data(),
                       theta_v.data(), x.data(), out.data()));
    return out;
}

/// qp.hpp:40-51
inline Vector recover_control(const Vector& z)
{
    if (z.size() % 2) throw std::invalid_argument("recover_control: odd length");
    const size_t n = z.size() / 2;
    Vector u(n);
    for (size_t i = 0; i < n; ++i) u[i] = z[i] - z[n + i];
    return u;
}

} // namespace optcon_b200
