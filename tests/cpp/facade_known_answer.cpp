// The reference's known-answer test (test_ipm.cpp:317-343) written against the
// C++ façade include/optcon_b200.hpp: a caller of the reference switches by
// changing the include and namespace. Exit code 0 = pass.
#include "optcon_b200.hpp"

#include <cmath>
#include <cstdio>

int main()
{
    using namespace optcon_b200;
    const Grid g(6);
    const int n = g.num_nodes();
    ControlProblem p;
    p.pde = PdeKind::poisson;
    p.alpha = 1e-4;
    p.beta = 1e-2;
    p.y_d.resize(n);
    for (int i = 0; i < n; ++i) {
        const double x = (i % g.nx() + 1) * g.h(), y = (i / g.nx() + 1) * g.h();
        p.y_d[i] = std::sin(M_PI * x) * std::sin(M_PI * y);
    }
    p.u_a.assign(n, -2.0);
    p.u_b.assign(n, 1.5);
    IpmParams params;
    params.sigma = 0.2;
    params.solver = SolverKind::gmres_pt;
    const IpmResult r = ipm_solve(build_qp(p, g), params);
    int fail = 0;
    if (!r.stats.converged) { std::puts("not converged"); ++fail; }
    if (r.stats.nli != 9) { std::printf("nli %d != 9\n", r.stats.nli); ++fail; }
    if (std::abs(r.state.mu - std::pow(0.2, 9)) > 1e-12 * std::pow(0.2, 9)) { std::puts("mu"); ++fail; }
    for (size_t k = 1; k < r.stats.iterations.size(); ++k) {
        const auto& it = r.stats.iterations[k];
        if (!(it.norm_xc <= 2.0 * it.mu) || !it.lin_converged) { std::puts("xi_c / lin"); ++fail; }
    }
    // reference error behaviour: heat through build_qp is rejected
    try {
        ControlProblem h = p;
        h.pde = PdeKind::heat;
        (void)build_qp(h, g);
        ++fail;
    } catch (const std::invalid_argument&) {
    }
    std::printf("facade known answer: nli=%d mu=%.6g av_li=%.3f J=%.12g %s\n", r.stats.nli,
                r.state.mu, r.stats.av_li, r.objective, fail ? "FAIL" : "ok");
    return fail;
}
