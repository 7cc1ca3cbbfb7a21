// Adapter at the reference's own plug-in point: an optcon::IpmModel whose
// newton_solve runs on the B200 (oc_newton_solve), driven by the reference's
// unmodified optcon::ipm_solve.
//
// The reference consumes the hot path through the IpmModel struct of
// std::function closures (ipm.hpp:70-93) built by make_steady_model
// (ipm.hpp:141, ipm.cpp:388-470) and make_spacetime_model (timedep.hpp:84,
// timedep.cpp:313-441); ipm_solve (ipm.cpp:270-341) calls
// model.newton_solve(theta, r1, r2, r3, params) once per interior-point
// iteration, and that call -- preconditioner setup (Chebyshev, m-hat, the
// multigrid hierarchies) plus the preconditioned Krylov solve -- is where the
// reference spends its time. The factories below
// return the reference's own model (its matvec closures and data untouched)
// with newton_solve bound to a device-resident copy of the same problem:
//
//     optcon::QpProblem qp = optcon::build_qp(problem, grid);              // reference
//     optcon::IpmModel  m  = optcon_b200::make_steady_model(qp, problem, grid);
//     optcon::IpmResult r  = optcon::ipm_solve(m, params);                 // reference loop
//
// to_b200() converts the reference's value types field by field. Needs the
// reference headers (optcon/ipm.hpp, optcon/timedep.hpp) on the include path
// and both libraries at link time (tests/cpp/ref_model_adapter.cpp).
#pragma once

#include "optcon_b200.hpp"

#include "optcon/ipm.hpp"
#include "optcon/timedep.hpp"

#include <memory>

namespace optcon_b200 {

/// qp.hpp:20-34 -> the façade's ControlProblem (same fields and meaning)
inline ControlProblem to_b200(const optcon::ControlProblem& p)
{
    ControlProblem b;
    switch (p.pde) {
    case optcon::PdeKind::poisson: b.pde = PdeKind::poisson; break;
    case optcon::PdeKind::convdiff: b.pde = PdeKind::convdiff; break;
    case optcon::PdeKind::heat: b.pde = PdeKind::heat; break;
    }
    b.eps = p.eps;
    b.tau = p.tau;
    b.horizon = p.horizon;
    b.alpha = p.alpha;
    b.beta = p.beta;
    b.y_d = p.y_d;
    b.f = p.f;
    b.u_a = p.u_a;
    b.u_b = p.u_b;
    b.y_a = p.y_a;
    b.y_b = p.y_b;
    if (p.observation)
        b.observation = ObservationRegion{p.observation->a1, p.observation->b1,
                                          p.observation->a2, p.observation->b2};
    return b;
}

/// grid.hpp:14-37
inline Grid to_b200(const optcon::Grid& g) { return Grid(g.level); }

/// ipm.hpp:17-32 (+ the device-only smoother choice; the reference's dense
/// verification solver has no device path and is rejected as the device
/// library rejects it: std::invalid_argument)
inline IpmParams to_b200(const optcon::IpmParams& p, int smoother = OC_SMOOTHER_AUTO)
{
    IpmParams b;
    b.alpha0 = p.alpha0;
    b.sigma = p.sigma;
    b.eps_p = p.eps_p;
    b.eps_d = p.eps_d;
    b.eps_c = p.eps_c;
    b.mu0 = p.mu0;
    b.max_iterations = p.max_iterations;
    b.linear_tol = p.linear_tol;
    b.linear_maxit = p.linear_maxit;
    b.cheb_steps = p.cheb_steps;
    b.mg_cycles = p.mg_cycles;
    b.mg_pre = p.mg_pre;
    b.mg_post = p.mg_post;
    switch (p.solver) {
    case optcon::SolverKind::gmres_pt: b.solver = SolverKind::gmres_pt; break;
    case optcon::SolverKind::minres_pd: b.solver = SolverKind::minres_pd; break;
    case optcon::SolverKind::gmres_ppi: b.solver = SolverKind::gmres_ppi; break;
    case optcon::SolverKind::dense:
        throw std::invalid_argument("newton_solve: the dense solver is a CPU verification path");
    }
    b.smoother = smoother;
    return b;
}

/// IpmModel::newton_solve on the device: uploads Theta and the right-hand
/// side, rebuilds the preconditioner for this Theta and runs the Krylov solve
/// (ipm.cpp:394-468 / timedep.cpp:335-439), returns dy, dz, dp and the
/// SolveReport (krylov.hpp:29-38) by value.
inline optcon::NewtonSolveResult device_newton_solve(const QpProblem& dev,
                                                     const optcon::ThetaBlocks& th,
                                                     const Vector& r1, const Vector& r2,
                                                     const Vector& r3,
                                                     const optcon::IpmParams& params,
                                                     int smoother)
{
    const size_t ny = static_cast<size_t>(dev.info().ny);
    if (r1.size() != ny || r2.size() != 2 * ny || r3.size() != ny || th.theta_w.size() != ny ||
        th.theta_v.size() != ny)
        throw std::invalid_argument("newton_solve: block size mismatch");
    const bool has_ty = dev.info().has_state_bounds && th.theta_y.size() == ny;
    const oc_ipm_params p = to_b200(params, smoother).c();
    optcon::NewtonSolveResult out;
    out.dy.resize(ny);
    out.dz.resize(2 * ny);
    out.dp.resize(ny);
    oc_solve_report rep{};
    check(oc_newton_solve(dev.get(), has_ty ? th.theta_y.data() : nullptr, th.theta_w.data(),
                          th.theta_v.data(), r1.data(), r2.data(), r3.data(), &p,
                          out.dy.data(), out.dz.data(), out.dp.data(), &rep));
    out.report.iterations = rep.iterations;
    out.report.relative_residual = rep.relative_residual;
    out.report.converged = rep.converged != 0;
    out.report.breakdown = rep.breakdown != 0;
    out.report.message = rep.message;
    return out;
}

/// make_steady_model (ipm.hpp:141) with the Newton solve on the device. The
/// reference QP must outlive the model (as for the reference's factory);
/// the device copy is owned by the model's closure.
inline optcon::IpmModel make_steady_model(const optcon::QpProblem& qp,
                                          const optcon::ControlProblem& problem,
                                          const optcon::Grid& grid,
                                          Context& ctx = default_context(),
                                          int smoother = OC_SMOOTHER_COLOR4)
{
    optcon::IpmModel m = optcon::make_steady_model(qp);
    auto dev = std::make_shared<QpProblem>(build_qp(to_b200(problem), to_b200(grid), ctx));
    if (dev->info().ny != m.ny) throw std::invalid_argument("make_steady_model: size mismatch");
    m.newton_solve = [dev, smoother](const optcon::ThetaBlocks& th, const Vector& r1,
                                     const Vector& r2, const Vector& r3,
                                     const optcon::IpmParams& params) {
        return device_newton_solve(*dev, th, r1, r2, r3, params, smoother);
    };
    return m;
}

/// make_spacetime_model (timedep.hpp:84) with the Newton solve on the device;
/// the device problem takes the system's (possibly overwritten) space-time y_d.
inline optcon::IpmModel make_spacetime_model(const optcon::SpaceTimeSystem& sys,
                                             const optcon::ControlProblem& problem,
                                             const optcon::Grid& grid,
                                             Context& ctx = default_context(),
                                             int smoother = OC_SMOOTHER_COLOR4)
{
    optcon::IpmModel m = optcon::make_spacetime_model(sys);
    ControlProblem bp = to_b200(problem);
    bp.y_d = sys.y_d;
    auto dev = std::make_shared<QpProblem>(assemble_spacetime(bp, to_b200(grid), ctx));
    if (dev->info().ny != m.ny) throw std::invalid_argument("make_spacetime_model: size mismatch");
    m.newton_solve = [dev, smoother](const optcon::ThetaBlocks& th, const Vector& r1,
                                     const Vector& r2, const Vector& r3,
                                     const optcon::IpmParams& params) {
        return device_newton_solve(*dev, th, r1, r2, r3, params, smoother);
    };
    return m;
}

} // namespace optcon_b200
