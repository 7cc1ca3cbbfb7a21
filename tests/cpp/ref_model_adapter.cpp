// The reference's UNMODIFIED ipm_solve (ipm.cpp:270-341) driven through its own
// plug-in point, IpmModel::newton_solve (ipm.hpp:70-93), bound to the device
// by optcon_b200::make_steady_model / make_spacetime_model
// (include/optcon_b200_ref.hpp), compared with the stock reference model
// (make_steady_model / make_spacetime_model with the reference's CPU Newton
// solve) on identical inputs.
//
// Cases: C1-style Poisson at level 6 (minres-pd and gmres-pt), C4-style
// convection-diffusion (eps 0.02, SUPG) at level 6, the state-box +
// partial-observation C3 style at level 5 with all Krylov solves converging
// (linear_maxit 3000; faithful lexicographic smoother), and space-time heat at
// level 4 with 8 steps.
// Pass: u and y within 1e-10 (relative 2-norm), the objective within 1e-10,
// the Newton count equal and every Newton solve converged.
//
// Built by oracle/Makefile (needs the reference headers and liboptcon_ref.so);
// run by tests/test_ref_adapter.py on a GPU. Prints one line per case.
#include "optcon_b200_ref.hpp"

#include "optcon/fem.hpp"
#include "optcon/grid.hpp"
#include "optcon/qp.hpp"

#include <cmath>
#include <cstdio>
#include <string>

namespace {

using optcon::Vector;

double rel(const Vector& a, const Vector& b)
{
    double d = 0.0, n = 0.0;
    for (size_t i = 0; i < a.size(); ++i) {
        d += (a[i] - b[i]) * (a[i] - b[i]);
        n += b[i] * b[i];
    }
    return n > 0 ? std::sqrt(d / n) : std::sqrt(d);
}

// four fixed sine modes, nodally interpolated (the bench's recipe with fixed draws)
Vector sine_modes(const optcon::Grid& g)
{
    const int nx = g.nx();
    const double h = g.h();
    const int k[4] = {1, 3, 2, 4}, l[4] = {2, 1, 4, 3};
    const double a[4] = {0.7, -0.4, 0.25, -0.55};
    Vector y(static_cast<size_t>(nx) * nx, 0.0);
    for (int j = 0; j < nx; ++j)
        for (int i = 0; i < nx; ++i)
            for (int m = 0; m < 4; ++m)
                y[static_cast<size_t>(j) * nx + i] +=
                    a[m] * std::sin(k[m] * M_PI * (i + 1) * h) * std::sin(l[m] * M_PI * (j + 1) * h);
    return y;
}

bool report(const std::string& name, const optcon::IpmResult& ref, const optcon::IpmResult& dev,
            double jref, double jdev)
{
    const double ru = rel(dev.u, ref.u), ry = rel(dev.state.y, ref.state.y);
    const double rj = std::abs(jdev - jref) / std::abs(jref);
    bool conv = dev.stats.converged;
    for (size_t i = 1; i < dev.stats.iterations.size(); ++i) conv = conv && dev.stats.iterations[i].lin_converged;
    const bool ok = ru <= 1e-10 && ry <= 1e-10 && rj <= 1e-10 && dev.stats.nli == ref.stats.nli && conv;
    std::printf("%s %s: rel_u=%.3e rel_y=%.3e rel_J=%.3e nli=%d/%d av_li=%.2f/%.2f converged=%d\n",
                ok ? "PASS" : "FAIL", name.c_str(), ru, ry, rj, dev.stats.nli, ref.stats.nli,
                dev.stats.av_li, ref.stats.av_li, conv ? 1 : 0);
    return ok;
}

bool steady_case(const std::string& name, optcon::ControlProblem p, int level,
                 optcon::IpmParams params, int smoother = OC_SMOOTHER_COLOR4)
{
    const optcon::Grid g(level);
    const size_t n = static_cast<size_t>(g.num_nodes());
    p.y_d = sine_modes(g);
    p.f.assign(n, 0.0);
    const optcon::QpProblem qp = optcon::build_qp(p, g);
    const optcon::IpmResult ref = optcon::ipm_solve(optcon::make_steady_model(qp), params);
    const optcon::IpmResult dev = optcon::ipm_solve(
        optcon_b200::make_steady_model(qp, p, g, optcon_b200::default_context(), smoother), params);
    return report(name, ref, dev, qp.objective(ref.state.y, ref.state.z),
                  qp.objective(dev.state.y, dev.state.z));
}

bool heat_case(const std::string& name, int level, int nt)
{
    const optcon::Grid g(level);
    const size_t n = static_cast<size_t>(g.num_nodes());
    optcon::ControlProblem p;
    p.pde = optcon::PdeKind::heat;
    p.tau = 1.0 / nt;
    p.alpha = 1e-3;
    p.beta = 1e-4;
    p.u_a.assign(n, -1.0);
    p.u_b.assign(n, 1.0);
    p.f.assign(n, 0.0);
    p.y_d = sine_modes(g);
    optcon::SpaceTimeSystem sys = optcon::assemble_spacetime(p, g);
    // time-decaying desired state: block k scaled by exp(-(k+1) tau)
    Vector yd(n * static_cast<size_t>(nt));
    for (int k = 0; k < nt; ++k)
        for (size_t i = 0; i < n; ++i) yd[static_cast<size_t>(k) * n + i] = p.y_d[i] * std::exp(-(k + 1) * p.tau);
    sys.y_d = yd;
    optcon::IpmParams params;
    params.solver = optcon::SolverKind::gmres_pt;
    const optcon::IpmResult ref = optcon::ipm_solve(optcon::make_spacetime_model(sys), params);
    const optcon::IpmResult dev =
        optcon::ipm_solve(optcon_b200::make_spacetime_model(sys, p, g), params);
    // objective through the model closures (no reference method for heat)
    const optcon::IpmModel m = optcon::make_spacetime_model(sys);
    auto J = [&](const optcon::IpmResult& r) {
        Vector d = r.state.y;
        for (size_t i = 0; i < d.size(); ++i) d[i] -= m.y_d[i];
        const Vector hd = m.hy(d), hz = m.hz(r.state.z);
        double v = 0.0;
        for (size_t i = 0; i < d.size(); ++i) v += 0.5 * d[i] * hd[i];
        for (size_t i = 0; i < hz.size(); ++i) v += 0.5 * r.state.z[i] * hz[i] + m.beta_grad[i] * r.state.z[i];
        return v;
    };
    return report(name, ref, dev, J(ref), J(dev));
}

} // namespace

int main()
{
    bool ok = true;
    try {
        {
            optcon::ControlProblem p;
            p.alpha = 1e-2;
            p.beta = 1e-3;
            const size_t n = static_cast<size_t>(optcon::Grid(6).num_nodes());
            p.u_a.assign(n, -2.0);
            p.u_b.assign(n, 2.0);
            optcon::IpmParams prm;
            prm.solver = optcon::SolverKind::minres_pd;
            ok = steady_case("C1 poisson l6 minres-pd", p, 6, prm) && ok;
            prm.solver = optcon::SolverKind::gmres_pt;
            ok = steady_case("C1 poisson l6 gmres-pt", p, 6, prm) && ok;
        }
        {
            optcon::ControlProblem p;
            p.pde = optcon::PdeKind::convdiff;
            p.eps = 0.02;
            p.alpha = 1e-4;
            p.beta = 1e-3;
            const size_t n = static_cast<size_t>(optcon::Grid(6).num_nodes());
            p.u_a.assign(n, -2.0);
            p.u_b.assign(n, 2.0);
            optcon::IpmParams prm;
            prm.solver = optcon::SolverKind::gmres_pt;
            ok = steady_case("C4 convdiff l6 gmres-pt", p, 6, prm) && ok;
        }
        {
            optcon::ControlProblem p;
            p.alpha = 1e-4;
            p.beta = 1e-3;
            const size_t n = static_cast<size_t>(optcon::Grid(5).num_nodes());
            p.u_a.assign(n, -2.0);
            p.u_b.assign(n, 2.0);
            p.y_a = Vector(n, -0.2);
            p.y_b = Vector(n, 0.3);
            p.observation = optcon::ObservationRegion(0.0, 0.5, 0.0, 1.0);
            optcon::IpmParams prm;
            prm.solver = optcon::SolverKind::gmres_ppi;
            prm.linear_maxit = 3000;
            // the state-constrained, partially observed system pins u only to
            // ~1e-9 at a 1e-10 Krylov residual (SURVEY §8c sensitivity table:
            // the reference's own variants differ by 1.5e-9): the faithful
            // lexicographic smoother reproduces the reference's preconditioner
            ok = steady_case("C3 state box + partial obs l5 gmres-ppi (lex)", p, 5, prm,
                             OC_SMOOTHER_LEX) && ok;
        }
        ok = heat_case("C5 heat l4 nt8 gmres-pt", 4, 8) && ok;
    } catch (const std::exception& e) {
        std::printf("FAIL exception: %s\n", e.what());
        return 2;
    }
    std::printf(ok ? "ALL PASS\n" : "SOME FAILED\n");
    return ok ? 0 : 1;
}
