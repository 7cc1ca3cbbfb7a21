/* C harness over the reference library compiled from /root/reference/proj/src
 * (TEST INFRASTRUCTURE ONLY — see oracle/README.md). Built by oracle/Makefile
 * into oracle/_ref/liboptcon_ref.so and driven from Python (oracle/ref.py) by
 * tests/ and by bench.py's CPU-baseline leg. Never linked by the product.
 *
 * Status codes: 0 ok, 1 std::invalid_argument, 2 std::runtime_error,
 * 3 other exception. ref_last_error() returns the exception text. */
#ifndef OPTCON_REF_HARNESS_H
#define OPTCON_REF_HARNESS_H

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    int pde;            /* 0 poisson, 1 convdiff, 2 heat */
    int level;
    double eps;         /* convdiff diffusion */
    double tau;         /* heat step */
    double horizon;     /* heat horizon */
    int quadrature;     /* heat: 0 rectangle, 1 trapezoid */
    double alpha, beta;
    const double* y_d;  /* n values, or n*nt for heat (space-time y_d) */
    long long y_d_len;
    const double* f;    /* nodal f, n values (NULL = zero) */
    const double* u_a;  /* n values */
    const double* u_b;
    const double* y_a;  /* NULL = no state box */
    const double* y_b;
    int has_obs;
    double obs[4];      /* a1, b1, a2, b2 */
} ref_problem_desc;

typedef struct {
    double alpha0, sigma, eps_p, eps_d, eps_c, mu0;
    int max_iterations;
    double linear_tol;
    int linear_maxit, cheb_steps, mg_cycles, mg_pre, mg_post;
    int solver; /* 0 gmres-pt, 1 minres-pd, 2 gmres-ppi, 3 dense,
                   10 heat minres-pd (harness composition of reference classes) */
} ref_params;

typedef struct {
    int k;
    double mu, norm_xp, norm_xd, norm_xc;
    int lin_iters;
    double lin_relres;
    int lin_converged;
    double newton_seconds;
} ref_record;

typedef struct {
    /* caller-allocated outputs (NULL to skip) */
    double *y, *z, *p, *lam_ya, *lam_yb, *lam_za, *lam_zb, *u;
    ref_record* records;
    int records_cap;
    /* filled */
    int n_records, nli, converged;
    double av_li, mu, objective, sparsity_pct, l1, nodal_sparsity_pct;
    long long total_lin;
    double newton_seconds, solve_seconds;
} ref_result;

const char* ref_last_error(void);
void* ref_problem_create(const ref_problem_desc* d);
void ref_problem_destroy(void* h);
/* n = spatial interior nodes, nt = time steps (1 for steady), ny = n*nt */
int ref_problem_sizes(void* h, int* n, int* nt, int* has_state_bounds);
int ref_ipm_solve(void* h, const ref_params* p, ref_result* r);
int ref_kkt_apply(void* h, const double* ty, const double* tw, const double* tv, const double* x,
                  double* out);
/* kind: 0 P_D, 1 P_T, 2 P_Pi, 3 heat P_T (timedep.cpp:396-426 composition),
         4 heat P_D (harness composition) */
int ref_precond_setup(void* h, const double* ty, const double* tw, const double* tv,
                      const ref_params* p);
int ref_precond_apply(void* h, int kind, const double* r, double* out);
/* Schur approximation inverse (precond.cpp:130-136) from the last setup */
int ref_schur_apply(void* h, const double* r, double* out);
/* wall seconds per KKT apply and per preconditioner apply, averaged over reps */
int ref_time_applies(void* h, int kind, int reps, const double* x, double* kkt_s, double* prec_s);
/* Bounded Krylov sample (bench.py's reference arm): prepare forms the first
 * IPM Newton system through the reference's ipm_solve and sets up the
 * preconditioner (solver as in ref_params; setup wall seconds returned); run
 * solves it with the reference's gmres (method 0) or minres (1) for at most
 * maxit iterations with preconditioner `kind` (ref_precond_apply kinds). */
int ref_newton_sample_prepare(void* h, const ref_params* p, double* setup_s);
int ref_newton_sample_run(void* h, int kind, int method, double tol, int maxit, int* iters,
                          double* relres, double* seconds);
/* objective of the steady QP (qp.cpp:112-121) or heat closures */
int ref_objective(void* h, const double* y, const double* z, double* out);
/* newton_rhs + build_theta + ipm_residuals on a given state (arrays as IpmState) */
int ref_ipm_pieces(void* h, const double* y, const double* z, const double* p,
                   const double* lam_ya, const double* lam_yb, const double* lam_za,
                   const double* lam_zb, double mu_state, double mu_rhs,
                   double* theta_y, double* theta_w, double* theta_v, double* r1, double* r2,
                   double* r3, double* norms3);

/* Assembled operators as 9 coefficient arrays (SW,S,SE,W,C,E,NW,N,NE; x fastest)
 * what: 0 mass, 1 poisson stiffness, 2 convdiff (eps, default wind, SUPG),
 *       3 partial mass (obs box), 4 lumped diagonal (writes n values) */
int ref_assemble9(int what, int level, double eps, const double* obs, double* coef);

/* Multigrid hierarchy over an explicit 9-diagonal fine matrix (multigrid.cpp) */
void* ref_mg_create(int level, const double* coef9, int rediscretize_convdiff, double eps,
                    int transpose_base);
int ref_mg_solve(void* mg, const double* rhs, int cycles, int pre, int post, double* out);
int ref_mg_depth(void* mg);
int ref_mg_level_matrix(void* mg, int k, double* coef9);
void ref_mg_destroy(void* mg);
int ref_gs_sweep(int level, const double* coef9, const double* b, double* x, int forward);

/* Chebyshev semi-iteration on scale*M + diag(extra) (chebyshev.cpp) */
int ref_cheb_apply(int level, double scale, const double* extra, int steps, const double* b,
                   double* x);

/* Krylov on an explicit 9-diagonal operator with a Jacobi preconditioner */
int ref_krylov_9diag(int method, int level, const double* coef9, const double* b, double tol,
                     int maxit, double* x, int* iters, double* relres);

#ifdef __cplusplus
}
#endif
#endif
