/* optcon-b200: C ABI of the B200-native (sm_100a, FP64) interior-point Newton
 * solve for L1-sparse, box-constrained PDE control (arXiv 1806.05896).
 *
 * This is the drop-in boundary beneath the reference's C++ solver API
 * (/root/reference/proj/include/optcon/ipm.hpp). Each entry point names the
 * reference interface it replaces. Plain pointers and sizes only; array
 * arguments may be host or device (cudaMalloc) pointers — the library detects
 * which. All vectors are FP64, interior nodes lexicographic with x fastest
 * (grid.hpp:31-36); saddle vectors are [y | w | v | p] (ipm.cpp:244-266).
 *
 * Status codes mirror the reference's exception classes:
 *   OC_OK 0, OC_INVALID_ARGUMENT 1 (std::invalid_argument),
 *   OC_RUNTIME_ERROR 2 (std::runtime_error), OC_CUDA_ERROR 3.
 * oc_last_error() returns the message of the last failure on this thread
 * (the reference's exception text where one exists).
 * There is no CPU fallback: without a CUDA device every call that computes
 * fails with OC_CUDA_ERROR. */
#ifndef OPTCON_B200_H
#define OPTCON_B200_H

#ifdef __cplusplus
extern "C" {
#endif

#define OC_OK 0
#define OC_INVALID_ARGUMENT 1
#define OC_RUNTIME_ERROR 2
#define OC_CUDA_ERROR 3

#define OC_ABI_VERSION 2

typedef struct oc_ctx oc_ctx;         /* one per host thread / stream */
typedef struct oc_problem oc_problem; /* device-resident QpProblem / SpaceTimeSystem */
typedef struct oc_mg oc_mg;           /* standalone multigrid hierarchy */

/* PdeKind (qp.hpp:16) */
enum { OC_PDE_POISSON = 0, OC_PDE_CONVDIFF = 1, OC_PDE_HEAT = 2 };
/* SolverKind (ipm.hpp:15); OC_SOLVER_DENSE is not offered on the device */
enum { OC_SOLVER_GMRES_PT = 0, OC_SOLVER_MINRES_PD = 1, OC_SOLVER_GMRES_PPI = 2 };
/* smoother: 4-colour symmetric Gauss-Seidel (parallel), the reference's
 * lexicographic Gauss-Seidel (multigrid.cpp:44-66) run as a skewed wavefront
 * (faithful mode), or AUTO (the IpmParams default): colour
 * sweeps while every Newton solve converges; a Newton solve that stops at
 * linear_maxit unconverged (krylov.cpp:133-212 cap: the iterate then depends
 * on the exact preconditioner) is discarded and re-solved with the
 * lexicographic smoother from the same Theta and right-hand side, which the
 * rest of the IPM solve keeps. */
enum { OC_SMOOTHER_COLOR4 = 0, OC_SMOOTHER_LEX = 1, OC_SMOOTHER_AUTO = 2 };
/* preconditioner kinds for oc_precond_apply */
enum { OC_PRECOND_PD = 0, OC_PRECOND_PT = 1, OC_PRECOND_PPI = 2 };

/* ControlProblem (qp.hpp:20-34) + Grid(level) + heat settings
 * (timedep.hpp:64-68). Replaces build_qp (qp.hpp:82) and
 * assemble_spacetime (timedep.hpp:68). */
typedef struct {
    int pde;             /* OC_PDE_* */
    int level;           /* grid level: h = 2^-level, (2^level-1)^2 interior nodes */
    double eps;          /* convection-diffusion diffusion */
    double tau;          /* heat time step */
    double horizon;      /* heat horizon T (tau must divide it) */
    int quadrature;      /* heat cost weights: 0 rectangle, 1 trapezoid */
    double alpha, beta;
    const double* y_d;   /* n (steady, heat constant-in-time) or n*nt (heat) values */
    long long y_d_len;
    const double* f;     /* nodal source, n values, or NULL for zero */
    const double* u_a;   /* control bounds, n values each */
    const double* u_b;
    const double* y_a;   /* state bounds, n values each, or NULL */
    const double* y_b;
    int has_obs;         /* partial observation box (ObservationRegion, grid.hpp:40-58) */
    double obs[4];       /* a1, b1, a2, b2 */
} oc_problem_desc;

/* IpmParams (ipm.hpp:17-32) */
typedef struct {
    double alpha0, sigma, eps_p, eps_d, eps_c, mu0;
    int max_iterations;
    double linear_tol;
    int linear_maxit, cheb_steps, mg_cycles, mg_pre, mg_post;
    int solver;          /* OC_SOLVER_* */
    int smoother;        /* OC_SMOOTHER_* */
    int gmres_restart;   /* 0 = full GMRES (reference); m > 0 restarts every m iterations */
} oc_ipm_params;

/* IterationRecord (ipm.hpp:44-53) + device time of the Newton solve */
typedef struct {
    int k;
    double mu, norm_xp, norm_xd, norm_xc;
    int lin_iters;
    double lin_relres;
    int lin_converged;
    double newton_ms;
} oc_iter_record;

/* IpmResult (ipm.hpp:100-105). Output arrays are caller-allocated (host or
 * device) and may be NULL: y, p, u, lam_ya, lam_yb (ny); z, lam_za, lam_zb (2ny). */
typedef struct {
    double *y, *z, *p, *lam_ya, *lam_yb, *lam_za, *lam_zb, *u;
    oc_iter_record* records;
    int records_cap;
    int n_records, nli, converged;
    double av_li, mu, objective;
    double sparsity_pct, l1;   /* sparsity_metric (qp.cpp:55-65) over interior nodes */
    double nodal_sparsity_pct; /* nodal_sparsity (bench.cpp:85-99), closed grid */
    long long total_lin;
    double solve_ms;           /* ipm_solve device time, initial point to exit */
    double newton_ms;          /* sum of Newton-solve device times */
    long long discarded_lin;   /* AUTO: Krylov iterations of capped colour-sweep solves
                                  that were re-solved (in solve_ms, not in total_lin) */
    int lex_from;              /* first Newton step (1-based) solved with the
                                  lexicographic smoother, 0 if none */
} oc_ipm_result;

/* SolveReport (krylov.hpp:29-38) */
typedef struct {
    int iterations;
    double relative_residual;
    int converged, breakdown;
    char message[96];
} oc_solve_report;

typedef struct {
    int n, nt;           /* spatial interior nodes, time blocks (1 steady) */
    long long ny;        /* n * nt */
    long long kkt_dim;   /* 4 * ny */
    int has_state_bounds, partial_observation, symmetric_k;
    int level;
    long long h2d_bytes;   /* bytes uploaded host->device by oc_problem_create */
} oc_problem_info;

const char* oc_last_error(void);
int oc_abi_version(void);

int oc_create(oc_ctx** ctx, int device);
void oc_destroy(oc_ctx* ctx);
int oc_synchronize(oc_ctx* ctx);

int oc_problem_create(oc_ctx* ctx, const oc_problem_desc* desc, oc_problem** out);
void oc_problem_destroy(oc_problem* prob);
int oc_problem_info_get(oc_problem* prob, oc_problem_info* info);

/* ipm_solve(make_steady_model(qp) | make_spacetime_model(sys), params)
 * (ipm.hpp:134,141; timedep.hpp:84) entirely on the device. */
int oc_default_params(oc_ipm_params* p);
int oc_ipm_solve(oc_problem* prob, const oc_ipm_params* params, oc_ipm_result* result);

/* make_saddle_operator(model, theta).apply (ipm.cpp:237-268): out = A x, 4ny. */
int oc_kkt_apply(oc_problem* prob, const double* theta_y, const double* theta_w,
                 const double* theta_v, const double* x, double* out);
/* Build the block preconditioners from Theta (Block11Approx + SchurApprox,
 * precond.cpp:110-169; PermutedPrecond :262-285; heat timedep.cpp:373-395).
 * theta_y may be NULL when there is no state box. */
int oc_precond_setup(oc_problem* prob, const double* theta_y, const double* theta_w,
                     const double* theta_v, const oc_ipm_params* params);
/* BlockDiagPrecond / BlockTriPrecond / PermutedPrecond ::apply
 * (precond.cpp:202-308), heat P_T (timedep.cpp:396-426). */
int oc_precond_apply(oc_problem* prob, int kind, const double* r, double* out);
/* SchurApprox::apply_inverse (precond.cpp:130-136) / TimeSchurApprox (timedep.cpp:268-311) */
int oc_schur_apply(oc_problem* prob, const double* r, double* out);
/* IpmModel::newton_solve (ipm.cpp:394-468): setup + Krylov on the device. */
int oc_newton_solve(oc_problem* prob, const double* theta_y, const double* theta_w,
                    const double* theta_v, const double* r1, const double* r2,
                    const double* r3, const oc_ipm_params* params, double* dy, double* dz,
                    double* dp, oc_solve_report* report);
/* build_theta + newton_rhs + ipm_residuals on a given state (ipm.cpp:32-143);
 * norms3 = RMS ||xi_p||, ||xi_d||, ||xi_c|| at barrier mu_state. */
int oc_ipm_pieces(oc_problem* prob, const double* y, const double* z, const double* p,
                  const double* lam_ya, const double* lam_yb, const double* lam_za,
                  const double* lam_zb, double mu_state, double mu_rhs, double* theta_y,
                  double* theta_w, double* theta_v, double* r1, double* r2, double* r3,
                  double* norms3);
/* QpProblem::objective (qp.cpp:112-121) */
int oc_objective(oc_problem* prob, const double* y, const double* z, double* out);
/* Device time (ms, CUDA events on the solver stream) of one KKT apply and one
 * preconditioner apply of `kind`, averaged over reps, at the last setup. */
int oc_time_applies(oc_problem* prob, int kind, int reps, double* kkt_ms, double* prec_ms);

/* MgHierarchy over an explicit 9-point operator (multigrid.hpp:43-64):
 * coef9 = 9 arrays of n values (SW,S,SE,W,C,E,NW,N,NE), host or device.
 * rediscretize: 0 plain Galerkin, 1 convdiff(eps) base per level,
 * 2 transposed convdiff base. smoother: OC_SMOOTHER_*. */
int oc_mg_create(oc_ctx* ctx, int level, const double* coef9, int rediscretize, double eps,
                 int smoother, oc_mg** out);
int oc_mg_solve(oc_mg* mg, const double* rhs, int cycles, int pre, int post, double* out);
int oc_mg_depth(oc_mg* mg);
int oc_mg_level_matrix(oc_mg* mg, int k, double* coef9);
void oc_mg_destroy(oc_mg* mg);
/* One smoothing sweep (forward/backward) of the configured smoother. */
int oc_mg_smooth(oc_mg* mg, const double* b, double* x, int forward);
/* ChebyshevSemiIteration(M(level), scale, extra, steps).apply(b) (chebyshev.cpp) */
int oc_cheb_apply(oc_ctx* ctx, int level, double scale, const double* extra, int steps,
                  const double* b, double* x);
/* Instrumentation (bench): kernel launches issued by this library so far;
 * per-launch CUDA-event profiling on the solver stream of fine-level smoothing
 * sweeps [0], KKT applies [1] and preconditioner applies [2]
 * (oc_profile_read returns summed ms and counts, then resets); and stream
 * events for timing a region on the solver stream (slots 0..7). */
long long oc_launch_count(void);
int oc_profile(oc_ctx* ctx, int enable);
int oc_profile_read(oc_ctx* ctx, double* ms4, long long* counts4);
int oc_event_record(oc_ctx* ctx, int slot);
int oc_event_elapsed(oc_ctx* ctx, int slot_a, int slot_b, double* ms);
/* elapsed ms from event slot_a of ctx_a to event slot_b of ctx_b (same device;
 * used to time concurrent solves on several contexts' streams) */
int oc_event_elapsed_between(oc_ctx* ctx_a, int slot_a, oc_ctx* ctx_b, int slot_b, double* ms);
/* Tuning aid: enable/disable %globaltimer phase stamps inside the cluster
 * multigrid bottom kernel and read the last launch's 64 stamps (CTA 0: 0..31,
 * CTA 1: 32..63; 0 = not reached). out64 may be NULL. */
int oc_debug_cluster_probes(int enable, unsigned long long* out64);
/* tuning aid: the dense 225 x 225 operator of the V-cycle below level 5 that the
   cluster bottom applies (row-major, batch element 0) */
int oc_debug_coarse_op(oc_mg* mg, int pre, int post, double* out);
/* Tuning knobs (process-wide): "sweep_tile" (-1 auto, 0: 64x32, 1: 32x32,
 * 2: 32x16, 3: 16x16, 4: 32x24 output tiles), "sweep_fuse" (1..5 smoothing sweeps per
 * launch, default 2), "cluster_bottom" (1: levels <= 7 in the 16-CTA cluster
 * kernel, 0: single-CTA bottom), "cluster_top8" (1: constant-stencil level-8
 * hierarchies, e.g. heat time blocks, solved whole in the cluster kernel),
 * "colour_split" (1: variable levels >= 511^2 sweep from a colour-split
 * coefficient copy), "cheb_block" (1: 5 Chebyshev steps per launch),
 * "fuse_norm" (1: a V-cycle's last sweep launch runs the divergence check),
 * "kkt_tiled" (1: the steady and the heat KKT apply from shared-memory halo
 * tiles), "heat_fork" (1: heat P_D's time-block substitution on the
 * high-priority side stream), "heat_chain" (1: each direction of the heat
 * time-block substitution as one chained cluster launch), "sweep_lean"
 * (variable tiled sweeps: 1 = 1/a_ii, 2 = 1/a_ii and b read in the colour
 * passes instead of staged, 3 = node records streamed into a shared-memory
 * ring by a producer warp's bulk copies; default 1),
 * "gmres_lazy_residual" (1: GMRES rebuilds x and forms the true residual only
 * once the residual norm it carries is within 1e3 of the tolerance, and at
 * every exit), "lex_pipeline" (1: the lexicographic sweeps of a smoothing phase run as a
 * pipelined batch of concurrent launches), "lex_bottom_top" (lexicographic
 * mode: top level of the single-CTA bottom
 * solver, 3..6, default 4; higher levels sweep as multi-CTA wavefronts),
 * "fuse_restrict" (1: a level's last pre-smoothing launch restricts its
 * residual), "mgs_persistent" (GMRES columns with j+1 >= value run their
 * modified Gram-Schmidt in one cooperative launch; default 8, 0 never).
 * Only launch shapes or layouts differ; results agree to rounding, and bit
 * for bit for every knob but the tile/fuse shapes and the cluster bottoms
 * ("kkt_tiled" regroups only the residual-norm partial sums). */
int oc_set_tuning(const char* name, int value);
/* Test hook: the lexicographic update's quotient (RN(1/d) product plus one
 * Markstein correction) against div.rn.f64 on n operand pairs (host or device
 * arrays); *mismatches = number of results that differ in any bit. */
int oc_debug_lex_div(oc_ctx* ctx, const double* num, const double* den, long long n,
                     unsigned long long* mismatches);
int oc_get_tuning(const char* name, int* value);

/* Q1 assembly into 9 coefficient arrays (fem.cpp:142-180; what: 0 mass,
 * 1 poisson, 2 convdiff(eps), 3 partial mass(obs), 4 lumped diagonal (n)). Host only. */
int oc_assemble9(int what, int level, double eps, const double* obs, double* coef);
/* The same assembly on the device (what 0..3; coef host or device, 9 n). */
int oc_assemble9_device(oc_ctx* ctx, int what, int level, double eps, const double* obs,
                        double* coef);

#ifdef __cplusplus
}
#endif
#endif
