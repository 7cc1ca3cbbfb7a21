// extern "C" boundary (include/optcon_b200.h): catches the library's C++
// exceptions and maps them to status codes mirroring the reference's
// exception classes (invalid_argument -> 1, runtime_error -> 2).
#include "assembly.hpp"
#include "solver.hpp"

#include <cstring>
#include <mutex>
#include <string>

// Lifetime: every problem and hierarchy holds its context's stream and pools
// (ocb::Ctx&), so a context is deleted only after its last child: oc_destroy
// on a context with live children marks it closing, and the last child's
// destroy deletes it (a façade context dying before its QpProblem).
struct oc_ctx {
    ocb::Ctx ctx;
    int children = 0;     // live problems and hierarchies (guarded by g_life)
    bool closing = false; // oc_destroy called while children were live
    explicit oc_ctx(int dev) : ctx(dev) {}
};

namespace {
std::mutex g_life;
void ctx_adopt(oc_ctx* c)
{
    std::lock_guard<std::mutex> lk(g_life);
    ++c->children;
}
void ctx_release(oc_ctx* c)
{
    bool del = false;
    {
        std::lock_guard<std::mutex> lk(g_life);
        del = --c->children == 0 && c->closing;
    }
    if (del) delete c;
}
} // namespace

struct oc_problem {
    std::unique_ptr<ocb::Problem> p;
    oc_ctx* owner = nullptr;
};

struct oc_mg {
    oc_ctx* owner = nullptr;
    ocb::Ctx* ctx = nullptr;
    int level = 0;
    ocb::DVec fine;
    std::vector<ocb::DVec> base;
    ocb::Hierarchy h;
    ocb::DVec t0, t1;
};

namespace {

thread_local std::string g_err;

template <typename F>
int guarded(F&& f)
{
    try {
        f();
        return OC_OK;
    } catch (const ocb::CudaFailure& e) {
        g_err = e.what();
        return OC_CUDA_ERROR;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return OC_INVALID_ARGUMENT;
    } catch (const std::runtime_error& e) {
        g_err = e.what();
        return OC_RUNTIME_ERROR;
    } catch (const std::exception& e) {
        g_err = e.what();
        return OC_RUNTIME_ERROR;
    }
}

void require(const void* p, const char* what)
{
    if (!p) throw ocb::InvalidArgument(std::string(what) + ": null argument");
}

} // namespace

extern "C" {

const char* oc_last_error(void) { return g_err.c_str(); }
int oc_abi_version(void) { return OC_ABI_VERSION; }

int oc_create(oc_ctx** out, int device)
{
    return guarded([&] {
        require(out, "oc_create");
        *out = new oc_ctx(device);
    });
}

void oc_destroy(oc_ctx* c)
{
    if (!c) return;
    {
        std::lock_guard<std::mutex> lk(g_life);
        if (c->children > 0) {
            c->closing = true; // the last problem / hierarchy deletes it
            return;
        }
    }
    delete c;
}

int oc_synchronize(oc_ctx* c)
{
    return guarded([&] {
        require(c, "oc_synchronize");
        c->ctx.sync();
    });
}

int oc_problem_create(oc_ctx* c, const oc_problem_desc* d, oc_problem** out)
{
    return guarded([&] {
        require(c, "oc_problem_create");
        require(d, "oc_problem_create");
        require(out, "oc_problem_create");
        auto p = std::make_unique<oc_problem>();
        p->p = std::make_unique<ocb::Problem>(c->ctx, *d);
        p->owner = c;
        ctx_adopt(c);
        *out = p.release();
    });
}

void oc_problem_destroy(oc_problem* p)
{
    if (!p) return;
    oc_ctx* owner = p->owner;
    delete p;
    if (owner) ctx_release(owner);
}

int oc_problem_info_get(oc_problem* p, oc_problem_info* info)
{
    return guarded([&] {
        require(p, "oc_problem_info_get");
        require(info, "oc_problem_info_get");
        *info = p->p->info();
    });
}

int oc_default_params(oc_ipm_params* p)
{
    return guarded([&] {
        require(p, "oc_default_params");
        // IpmParams defaults (ipm.hpp:17-32)
        p->alpha0 = 0.995;
        p->sigma = 0.2;
        p->eps_p = p->eps_d = p->eps_c = 1e-6;
        p->mu0 = 1.0;
        p->max_iterations = 100;
        p->linear_tol = 1e-10;
        p->linear_maxit = 200;
        p->cheb_steps = 20;
        p->mg_cycles = 3;
        p->mg_pre = 5;
        p->mg_post = 5;
        p->solver = OC_SOLVER_GMRES_PT;
        p->smoother = OC_SMOOTHER_AUTO;
        p->gmres_restart = 0;
    });
}

int oc_ipm_solve(oc_problem* p, const oc_ipm_params* params, oc_ipm_result* r)
{
    return guarded([&] {
        require(p, "oc_ipm_solve");
        require(params, "oc_ipm_solve");
        require(r, "oc_ipm_solve");
        p->p->ipm_solve(*params, r);
    });
}

int oc_kkt_apply(oc_problem* p, const double* ty, const double* tw, const double* tv,
                 const double* x, double* out)
{
    return guarded([&] {
        require(p, "oc_kkt_apply");
        require(tw, "oc_kkt_apply");
        require(tv, "oc_kkt_apply");
        require(x, "oc_kkt_apply");
        require(out, "oc_kkt_apply");
        ocb::Problem& P = *p->p;
        const size_t n4 = 4 * (size_t)P.P.ny;
        P.set_theta(ty, tw, tv);
        ocb::DVec xin(n4), o(n4);
        ocb::copy_any(P.ctx, xin.get(), x, n4 * 8);
        P.kkt(xin.get(), o.get());
        ocb::copy_any(P.ctx, out, o.get(), n4 * 8);
        P.ctx.sync();
    });
}

int oc_precond_setup(oc_problem* p, const double* ty, const double* tw, const double* tv,
                     const oc_ipm_params* params)
{
    return guarded([&] {
        require(p, "oc_precond_setup");
        require(params, "oc_precond_setup");
        ocb::Problem& P = *p->p;
        P.set_theta(ty, tw, tv);
        const oc_problem_info info = P.info();
        int kind = params->solver == OC_SOLVER_GMRES_PPI ? OC_PRECOND_PPI
                   : params->solver == OC_SOLVER_MINRES_PD ? OC_PRECOND_PD
                                                           : OC_PRECOND_PT;
        if (info.partial_observation && kind != OC_PRECOND_PPI)
            throw ocb::InvalidArgument(kind == OC_PRECOND_PD
                                           ? "minres-pd requires a nonsingular (1,1) block"
                                           : "gmres-pt requires a nonsingular (1,1) block");
        P.setup_precond(kind, *params);
        P.ctx.sync();
    });
}

int oc_precond_apply(oc_problem* p, int kind, const double* r, double* out)
{
    return guarded([&] {
        require(p, "oc_precond_apply");
        require(r, "oc_precond_apply");
        require(out, "oc_precond_apply");
        ocb::Problem& P = *p->p;
        const size_t n4 = 4 * (size_t)P.P.ny;
        ocb::DVec rin(n4), o(n4);
        ocb::copy_any(P.ctx, rin.get(), r, n4 * 8);
        P.precond_apply(kind, rin.get(), o.get());
        ocb::copy_any(P.ctx, out, o.get(), n4 * 8);
        P.ctx.sync();
    });
}

int oc_schur_apply(oc_problem* p, const double* r, double* out)
{
    return guarded([&] {
        require(p, "oc_schur_apply");
        ocb::Problem& P = *p->p;
        const size_t n = (size_t)P.P.ny;
        ocb::DVec rin(n), o(n);
        ocb::copy_any(P.ctx, rin.get(), r, n * 8);
        P.schur_apply(rin.get(), o.get());
        ocb::copy_any(P.ctx, out, o.get(), n * 8);
        P.ctx.sync();
    });
}

int oc_newton_solve(oc_problem* p, const double* ty, const double* tw, const double* tv,
                    const double* r1, const double* r2, const double* r3,
                    const oc_ipm_params* params, double* dy, double* dz, double* dp,
                    oc_solve_report* report)
{
    return guarded([&] {
        require(p, "oc_newton_solve");
        require(params, "oc_newton_solve");
        ocb::Problem& P = *p->p;
        const size_t n = (size_t)P.P.ny;
        P.set_theta(ty, tw, tv);
        ocb::DVec rhs(4 * n), x(4 * n);
        ocb::copy_any(P.ctx, rhs.get(), r1, n * 8);
        ocb::copy_any(P.ctx, rhs.get() + n, r2, 2 * n * 8);
        ocb::copy_any(P.ctx, rhs.get() + 3 * n, r3, n * 8);
        const oc_solve_report rep = P.newton_solve(*params, rhs.get(), x.get());
        if (dy) ocb::copy_any(P.ctx, dy, x.get(), n * 8);
        if (dz) ocb::copy_any(P.ctx, dz, x.get() + n, 2 * n * 8);
        if (dp) ocb::copy_any(P.ctx, dp, x.get() + 3 * n, n * 8);
        P.ctx.sync();
        if (report) *report = rep;
    });
}

int oc_ipm_pieces(oc_problem* p, const double* y, const double* z, const double* pv,
                  const double* lya, const double* lyb, const double* lza, const double* lzb,
                  double mu_state, double mu_rhs, double* ty, double* tw, double* tv, double* r1,
                  double* r2, double* r3, double* norms3)
{
    return guarded([&] {
        require(p, "oc_ipm_pieces");
        p->p->ipm_pieces(y, z, pv, lya, lyb, lza, lzb, mu_state, mu_rhs, ty, tw, tv, r1, r2, r3,
                         norms3);
    });
}

int oc_objective(oc_problem* p, const double* y, const double* z, double* out)
{
    return guarded([&] {
        require(p, "oc_objective");
        require(out, "oc_objective");
        *out = p->p->objective(y, z);
    });
}

int oc_time_applies(oc_problem* p, int kind, int reps, double* kkt_ms, double* prec_ms)
{
    return guarded([&] {
        require(p, "oc_time_applies");
        if (reps < 1) throw ocb::InvalidArgument("oc_time_applies: reps must be >= 1");
        p->p->time_applies(kind, reps, kkt_ms, prec_ms);
    });
}

int oc_mg_create(oc_ctx* c, int level, const double* coef9, int rediscretize, double eps,
                 int smoother, oc_mg** out)
{
    return guarded([&] {
        require(c, "oc_mg_create");
        require(coef9, "oc_mg_create");
        require(out, "oc_mg_create");
        if (level < 3) throw ocb::InvalidArgument("MgHierarchy: fine level must be >= 3");
        auto m = std::make_unique<oc_mg>();
        m->ctx = &c->ctx;
        m->level = level;
        const long long n = ocb::level_n(level);
        m->fine.resize(9 * (size_t)n);
        ocb::copy_any(c->ctx, m->fine.get(), coef9, 9 * (size_t)n * 8);
        m->h.allocate(level, 1, smoother);
        ocb::Op9 f{};
        f.nx = ocb::level_nx(level);
        f.coef = m->fine.get();
        f.cscale = 1.0;
        if (rediscretize) {
            std::vector<const double*> b;
            for (int l = level; l >= 2; --l) {
                std::vector<double> a = ocb::assemble_convdiff9(l, eps, true);
                if (rediscretize == 2) a = ocb::transpose9(a, l);
                m->base.emplace_back(a.size());
                ocb::copy_any(c->ctx, m->base.back().get(), a.data(), a.size() * 8);
                c->ctx.sync();
            }
            for (auto& v : m->base) b.push_back(v.get());
            m->h.build_rediscretized(c->ctx, f, b);
        } else {
            m->h.build(c->ctx, f);
        }
        m->t0.resize((size_t)n);
        m->t1.resize((size_t)n);
        c->ctx.sync();
        m->owner = c;
        ctx_adopt(c);
        *out = m.release();
    });
}

int oc_mg_solve(oc_mg* m, const double* rhs, int cycles, int pre, int post, double* out)
{
    return guarded([&] {
        require(m, "oc_mg_solve");
        const long long n = ocb::level_n(m->level);
        ocb::copy_any(*m->ctx, m->t0.get(), rhs, (size_t)n * 8);
        ocb::DevArray<int> flags(1);
        cudaMemsetAsync(flags.get(), 0, sizeof(int), m->ctx->stream);
        ocb::MgParams p;
        p.cycles = cycles;
        p.pre = pre;
        p.post = post;
        m->h.solve(*m->ctx, m->t0.get(), m->t1.get(), p, 0, flags.get());
        ocb::copy_any(*m->ctx, out, m->t1.get(), (size_t)n * 8);
        cudaMemcpyAsync(m->ctx->hflags, flags.get(), sizeof(int), cudaMemcpyDeviceToHost,
                        m->ctx->stream);
        m->ctx->sync();
        if (m->ctx->hflags[0] & ocb::kErrMgDiverged)
            throw ocb::RuntimeError("MgHierarchy::solve: residual growth, cycle diverged");
        if (m->ctx->hflags[0] & ocb::kErrLexStall)
            throw ocb::RuntimeError("gauss_seidel_sweep: wavefront hand-off stalled");
    });
}

int oc_mg_depth(oc_mg* m) { return m ? m->h.depth() : -1; }

int oc_mg_level_matrix(oc_mg* m, int k, double* coef9)
{
    return guarded([&] {
        require(m, "oc_mg_level_matrix");
        if (k < 0 || k > m->h.depth()) throw ocb::InvalidArgument("oc_mg_level_matrix: bad level");
        const ocb::Op9 a = m->h.level_op(k, 0);
        ocb::copy_any(*m->ctx, coef9, a.coef, 9 * (size_t)m->h.level_n(k) * 8);
        m->ctx->sync();
    });
}

int oc_mg_smooth(oc_mg* m, const double* b, double* x, int forward)
{
    return guarded([&] {
        require(m, "oc_mg_smooth");
        const long long n = ocb::level_n(m->level);
        ocb::copy_any(*m->ctx, m->t0.get(), b, (size_t)n * 8);
        ocb::copy_any(*m->ctx, m->t1.get(), x, (size_t)n * 8);
        m->h.smooth(*m->ctx, m->t0.get(), m->t1.get(), forward != 0, 0);
        ocb::copy_any(*m->ctx, x, m->t1.get(), (size_t)n * 8);
        m->ctx->sync();
    });
}

void oc_mg_destroy(oc_mg* m)
{
    if (!m) return;
    if (m->ctx) cudaStreamSynchronize(m->ctx->stream);
    oc_ctx* owner = m->owner;
    delete m;
    if (owner) ctx_release(owner);
}

int oc_cheb_apply(oc_ctx* c, int level, double scale, const double* extra, int steps,
                  const double* b, double* x)
{
    return guarded([&] {
        require(c, "oc_cheb_apply");
        if (steps < 1) throw ocb::InvalidArgument("chebyshev: steps must be >= 1");
        ocb::Ctx& cx = c->ctx;
        const int nx = ocb::level_nx(level);
        const long long n = (long long)nx * nx;
        double cM[9];
        ocb::stencil9(0, level, cM);
        ocb::ProbDev P{};
        P.nx = nx;
        P.ns = n;
        P.nt = 1;
        P.ny = n;
        P.heat = 1; // scale applied as the per-block weight tau*w_0 = scale
        P.tau = scale;
        P.M.nx = nx;
        P.M.cscale = 1.0;
        for (int d = 0; d < 9; ++d) P.M.c[d] = cM[d];
        const double one = 1.0;
        ocb::DVec qw(1), bb((size_t)n), e, out((size_t)n), g((size_t)n), r0((size_t)n),
            r1((size_t)n), r2((size_t)n);
        ocb::copy_any(cx, qw.get(), &one, 8);
        P.qw = qw.get();
        ocb::copy_any(cx, bb.get(), b, (size_t)n * 8);
        if (extra) {
            e.resize((size_t)n);
            ocb::copy_any(cx, e.get(), extra, (size_t)n * 8);
        }
        ocb::ChebWork w{g.get(), r0.get(), r1.get(), r2.get()};
        ocb::launch_chebyshev(cx.stream, P, bb.get(), extra ? e.get() : nullptr, steps, w,
                              out.get());
        ocb::copy_any(cx, x, out.get(), (size_t)n * 8);
        cx.sync();
    });
}

long long oc_launch_count(void) { return ocb::launch_count(); }

int oc_set_tuning(const char* name, int value)
{
    return guarded([&] {
        require(name, "oc_set_tuning");
        const std::string k = name;
        if (k == "sweep_tile") ocb::g_sweep_tile = value;
        else if (k == "sweep_fuse") ocb::g_sweep_fuse = value;
        else if (k == "cluster_bottom") ocb::g_cluster_bottom = value;
        else if (k == "cluster_top8") ocb::g_cluster_top8 = value;
        else if (k == "colour_split") ocb::g_colour_split = value;
        else if (k == "sweep_lean") ocb::g_sweep_lean = value;
        else if (k == "mgs_persistent") ocb::g_mgs_persistent = value;
        else if (k == "cheb_block") ocb::g_cheb_block = value;
        else if (k == "fuse_norm") ocb::g_fuse_norm = value;
        else if (k == "fuse_restrict") ocb::g_fuse_restrict = value;
        else if (k == "kkt_tiled") ocb::g_kkt_tiled = value;
        else if (k == "heat_fork") ocb::g_heat_fork = value;
        else if (k == "heat_chain") ocb::g_heat_chain = value;
        else if (k == "lex_pipeline") ocb::g_lex_pipeline = value;
        else if (k == "gmres_lazy_residual") ocb::g_gmres_lazy_residual = value;
        else if (k == "lex_start") ocb::g_lex_start = value < 17 ? 17 : value;
        else if (k == "lex_bottom_top") ocb::g_lex_bottom_top = value < 3 ? 3 : (value > 6 ? 6 : value);
        else throw ocb::InvalidArgument("oc_set_tuning: unknown knob " + k);
        // captured preconditioner graphs hold the old launch shapes: drop them
        ocb::g_tuning_gen.fetch_add(1);
    });
}

int oc_get_tuning(const char* name, int* value)
{
    return guarded([&] {
        require(name, "oc_get_tuning");
        require(value, "oc_get_tuning");
        const std::string k = name;
        if (k == "sweep_tile") *value = ocb::g_sweep_tile;
        else if (k == "sweep_fuse") *value = ocb::g_sweep_fuse;
        else if (k == "cluster_bottom") *value = ocb::g_cluster_bottom;
        else if (k == "cluster_top8") *value = ocb::g_cluster_top8;
        else if (k == "colour_split") *value = ocb::g_colour_split;
        else if (k == "sweep_lean") *value = ocb::g_sweep_lean;
        else if (k == "mgs_persistent") *value = ocb::g_mgs_persistent;
        else if (k == "cheb_block") *value = ocb::g_cheb_block;
        else if (k == "fuse_norm") *value = ocb::g_fuse_norm;
        else if (k == "fuse_restrict") *value = ocb::g_fuse_restrict;
        else if (k == "kkt_tiled") *value = ocb::g_kkt_tiled;
        else if (k == "heat_fork") *value = ocb::g_heat_fork;
        else if (k == "heat_chain") *value = ocb::g_heat_chain;
        else if (k == "lex_pipeline") *value = ocb::g_lex_pipeline;
        else if (k == "gmres_lazy_residual") *value = ocb::g_gmres_lazy_residual;
        else if (k == "lex_start") *value = ocb::g_lex_start;
        else if (k == "lex_bottom_top") *value = ocb::g_lex_bottom_top;
        else throw ocb::InvalidArgument("oc_get_tuning: unknown knob " + k);
    });
}

int oc_debug_coarse_op(oc_mg* m, int pre, int post, double* out)
{
    return guarded([&] {
        require(m, "oc_debug_coarse_op");
        m->h.ensure_coarse_op(*m->ctx, pre, post);
        const double* d = m->h.coarse_op();
        if (!d) throw ocb::InvalidArgument("oc_debug_coarse_op: hierarchy has no cluster bottom");
        ocb::copy_any(*m->ctx, out, d, (size_t)ocb::kCoarseOpN * ocb::kCoarseOpN * 8);
        m->ctx->sync();
        ocb::cuda_check(cudaGetLastError(), "coarse operator");
    });
}

int oc_debug_lex_div(oc_ctx* c, const double* num, const double* den, long long n,
                     unsigned long long* mismatches)
{
    return guarded([&] {
        require(c, "oc_debug_lex_div");
        require(mismatches, "oc_debug_lex_div");
        ocb::DVec a((size_t)n), b((size_t)n);
        ocb::DevArray<unsigned long long> bad(1);
        ocb::copy_any(c->ctx, a.get(), num, (size_t)n * 8);
        ocb::copy_any(c->ctx, b.get(), den, (size_t)n * 8);
        cudaMemsetAsync(bad.get(), 0, sizeof(unsigned long long), c->ctx.stream);
        ocb::launch_lex_div_check(c->ctx.stream, a.get(), b.get(), n, bad.get());
        ocb::copy_any(c->ctx, mismatches, bad.get(), sizeof(unsigned long long));
        c->ctx.sync();
        ocb::cuda_check(cudaGetLastError(), "lex division check");
    });
}

int oc_debug_cluster_probes(int enable, unsigned long long* out64)
{
    // enable >= 2: the lexicographic sweep's stamps instead (out64: 512 words)
    if (enable >= 2) return guarded([&] { ocb::lex_probes(enable - 2, out64); });
    return guarded([&] { ocb::cluster_probes(enable, out64); });
}

int oc_profile(oc_ctx* c, int enable)
{
    return guarded([&] {
        require(c, "oc_profile");
        c->ctx.prof.on = enable != 0;
    });
}

int oc_profile_read(oc_ctx* c, double* ms4, long long* counts4)
{
    return guarded([&] {
        require(c, "oc_profile_read");
        require(ms4, "oc_profile_read");
        require(counts4, "oc_profile_read");
        c->ctx.prof.read(ms4, counts4);
    });
}

int oc_event_record(oc_ctx* c, int slot)
{
    return guarded([&] {
        require(c, "oc_event_record");
        if (slot < 0 || slot >= 8) throw ocb::InvalidArgument("oc_event_record: slot out of range");
        ocb::cuda_check(cudaEventRecord(c->ctx.user_ev[slot], c->ctx.stream), "cudaEventRecord");
    });
}

int oc_event_elapsed(oc_ctx* c, int a, int b, double* ms)
{
    return guarded([&] {
        require(c, "oc_event_elapsed");
        require(ms, "oc_event_elapsed");
        if (a < 0 || a >= 8 || b < 0 || b >= 8)
            throw ocb::InvalidArgument("oc_event_elapsed: slot out of range");
        ocb::cuda_check(cudaEventSynchronize(c->ctx.user_ev[b]), "cudaEventSynchronize");
        float t = 0.f;
        ocb::cuda_check(cudaEventElapsedTime(&t, c->ctx.user_ev[a], c->ctx.user_ev[b]),
                        "cudaEventElapsedTime");
        *ms = t;
    });
}

int oc_event_elapsed_between(oc_ctx* ca, int a, oc_ctx* cb, int b, double* ms)
{
    return guarded([&] {
        require(ca, "oc_event_elapsed_between");
        require(cb, "oc_event_elapsed_between");
        require(ms, "oc_event_elapsed_between");
        if (a < 0 || a >= 8 || b < 0 || b >= 8)
            throw ocb::InvalidArgument("oc_event_elapsed_between: slot out of range");
        ocb::cuda_check(cudaEventSynchronize(ca->ctx.user_ev[a]), "cudaEventSynchronize");
        ocb::cuda_check(cudaEventSynchronize(cb->ctx.user_ev[b]), "cudaEventSynchronize");
        float t = 0.f;
        ocb::cuda_check(cudaEventElapsedTime(&t, ca->ctx.user_ev[a], cb->ctx.user_ev[b]),
                        "cudaEventElapsedTime");
        *ms = t;
    });
}

int oc_assemble9(int what, int level, double eps, const double* obs, double* coef)
{
    return guarded([&] {
        require(coef, "oc_assemble9");
        std::vector<double> a;
        switch (what) {
        case 0: a = ocb::assemble_mass9(level); break;
        case 1: a = ocb::assemble_poisson9(level); break;
        case 2: a = ocb::assemble_convdiff9(level, eps, true); break;
        case 3: require(obs, "oc_assemble9"); a = ocb::assemble_partial_mass9(level, obs); break;
        case 4: a = ocb::lumped_diag(level); break;
        default: throw ocb::InvalidArgument("oc_assemble9: unknown operator");
        }
        std::memcpy(coef, a.data(), a.size() * sizeof(double));
    });
}

int oc_assemble9_device(oc_ctx* c, int what, int level, double eps, const double* obs, double* coef)
{
    return guarded([&] {
        require(c, "oc_assemble9_device");
        require(coef, "oc_assemble9_device");
        if (level < 1 || level > 14) throw ocb::InvalidArgument("Grid: level out of range");
        if (what < 0 || what > 3) throw ocb::InvalidArgument("oc_assemble9: unknown operator");
        if (what == 2 && eps <= 0.0) throw ocb::InvalidArgument("assemble_convdiff: eps must be positive");
        if (what == 3) require(obs, "oc_assemble9_device");
        const size_t m = 9 * (size_t)ocb::level_n(level);
        ocb::DVec d(m);
        ocb::launch_assemble9(c->ctx.stream, what, level, eps, obs, d.get());
        ocb::copy_any(c->ctx, coef, d.get(), m * sizeof(double));
        c->ctx.sync();
    });
}

} // extern "C"
