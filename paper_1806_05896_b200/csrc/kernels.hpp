// Host-callable launchers for the sm_100a kernels (FP64, bandwidth-bound).
// Every launcher enqueues on the given stream and never synchronises.
#pragma once

#include "oc_common.cuh"

#include <atomic>

namespace ocb {

// Count of kernel launches issued by this library (bench "gpu_launches").
void note_launch();
int active_contexts(); // live oc_ctx objects in this process (tile-shape heuristic)
void add_launches(long long k); // graph replays count their kernel nodes
long long launch_count();

// ---------------------------------------------------------------- multigrid
struct MgLevelDev {
    Op9 op;          // level operator (fine: constant stencil + diag, coarse: 9 arrays)
    double* x;       // level iterate (coarse levels only; fine uses caller buffers)
    double* b;       // level right-hand side (coarse levels only)
};

constexpr int kBottomMaxLevels = 7;   // levels 2..8 at most (cluster kernel with a level-8 top)
constexpr int kBottomTopLevel = 6;    // grid levels <= this run inside one CTA
extern std::atomic<int> g_lex_bottom_top; // lexicographic mode: top level of the single-CTA bottom (4)
extern std::atomic<int> g_lex_start;      // lexicographic sweep: band start column of the band above

struct BottomArgs {
    int nlev;                          // number of levels handled (top .. level 2)
    int lex;                           // lexicographic (reference) smoother instead of 4-colour
    Op9 ops[kBottomMaxLevels];         // [0] = top level of the bottom solver
    const double* lu;                  // 9x9 LU of the level-2 matrix (column-major)
    const int* perm;
    const double* cop;                 // cluster kernel: dense levels <= 4 cycle operator (225 x 225)
};

// k_mg_tiled.cu: the smoothing sweep and the fused residual + restriction
// (bc = R (b - A x), R = P^T; also zeroes xc), tiled for the multi-CTA levels:
// `ns` fused sweeps per launch (1..5); g_sweep_tile overrides the tile choice.
// process-wide tuning knobs (oc_set_tuning), read by every solving thread
extern std::atomic<int> g_sweep_tile;
extern std::atomic<int> g_cluster_bottom; // 1: levels <= 7 in the cluster kernel (default), 0: single-CTA bottom
extern std::atomic<int> g_sweep_fuse;     // sweeps per launch in the V-cycle (1..5, temporal blocking)
extern std::atomic<int> g_cluster_top8;   // 1: constant-stencil level-8 hierarchies run whole in the cluster kernel
// inv = 1 / diag(A) precomputed per level (launch_inv_diag).
// With part != nullptr the launch also runs the divergence check of
// launch_residual_norm_check on its result when it can (<= 2 sweeps, grid <=
// kNormBlocks); with bc != nullptr it also does launch_resid_restrict_tiled's
// work (bc = R (b - A x), xc = 0; <= 2 sweeps). Returns whether it fused.
bool launch_sweep_tiled(cudaStream_t s, const Op9& A, const double* b, const double* inv,
                        const double* x, double* xo, bool forward, bool zero_init,
                        const double* ec, int ns, double* part = nullptr,
                        unsigned* counter = nullptr, double* state = nullptr, int* flags = nullptr,
                        double* bc = nullptr, double* xc = nullptr);
// (dfull != nullptr: also the diagonal values themselves)
void launch_inv_diag(cudaStream_t s, const Op9& A, double* inv, int batch, long long fcs,
                     long long fds, double* dfull = nullptr);
// colour-split copy (Op9::csplit) of a variable operator's 8 off-diagonal planes
extern std::atomic<int> g_mgs_persistent; // GMRES columns j+1 >= this use the persistent MGS launch (0: never)
extern std::atomic<int> g_sweep_lean;   // variable tiled sweeps: 1 = 1/a_ii, 2 = 1/a_ii and b read in the passes, not staged
extern std::atomic<int> g_colour_split; // 1: the fine level of >= 1023^2 hierarchies sweeps from it
void launch_colour_split(cudaStream_t s, int nx, const double* coef, const double* diag, double* out);
constexpr int kSplitRecordWords = 10; // words per node of the colour-split copy
void launch_resid_restrict_tiled(cudaStream_t s, const Op9& A, const double* b, const double* x,
                                 double* bc, double* xc);
// x += P ec
void launch_prolong_add(cudaStream_t s, int nx, const double* ec, double* x);
// Divergence check of MgHierarchy::solve (multigrid.cpp:141-157) in one launch:
// res = ||b - A x|| (kRedBlocks partials in part, summed in a fixed order by the
// block that finishes last); flag if res > 10 state[0]; state[0] = res.
// part: kNormBlocks doubles.
// counter: one zero-initialised unsigned per hierarchy (reset by the kernel).
void launch_residual_norm_check(cudaStream_t s, const Op9& A, const double* b, const double* x,
                                double* part, unsigned* counter, double* state, int* flags);
// state[0] = ||b||  (initial "previous residual")
void launch_norm_init(cudaStream_t s, const double* b, long long n, double* part,
                      unsigned* counter, double* state);
// Galerkin R A P into 9 coarse arrays; if base != nullptr the result is base + RAP.
// batch > 1 (heat blocks): fine coef/diag and coarse arrays advance by the given strides.
// If rem_out != nullptr the bare R A P is also written there (rediscretised chain).
void launch_rap(cudaStream_t s, const Op9& fine, double* coarse, const double* base,
                double* rem_out, int batch, long long fine_coef_stride,
                long long fine_diag_stride, long long coarse_stride);
// Fine remainder of a rediscretised hierarchy (multigrid.cpp:86-88):
// rem9 = fine - base over all 9 entries (fine may be constant + diag or arrays).
void launch_remainder9(cudaStream_t s, const Op9& fine, const double* base9, double* rem9);
// 9x9 coarse LU with partial pivoting (dense_eig.cpp:87-121 semantics)
void launch_coarse_lu(cudaStream_t s, const double* coef9, double* lu, int* perm, int batch);
// whole V-cycle below (and including) the bottom top level in one CTA
void launch_bottom(cudaStream_t s, const BottomArgs& a, const double* b, double* x, int cycles,
                   int pre, int post, bool check, double* state, int* flags);

// k_mg_lex.cu: one lexicographic Gauss-Seidel sweep in place (the reference
// smoother, multigrid.cpp:44-66) as a skewed wavefront; inv = 1/diag(A);
// mbox = ceil(nx/32) * nx doubles holding kLexSentinel (restored on return).
// dfull = a_ii (the CSR diagonal value: centre coefficient + added diagonal).
void launch_gs_lex(cudaStream_t s, const Op9& A, const double* b, const double* inv,
                   const double* dfull, double* x, bool forward, double* mbox, int* flags,
                   const int* prog_prev = nullptr, int* prog_out = nullptr);
// Pipelined batch of lexicographic sweeps (k_mg_lex.cu, LexArgs::prog_*): up to
// kLexPipe sweeps of one level in flight, each launch with its own mailbox set.
constexpr int kLexPipe = 5;
extern std::atomic<int> g_lex_pipeline;
// test hook: mismatches of the lexicographic update's quotient vs div.rn.f64
void launch_lex_div_check(cudaStream_t s, const double* num, const double* den, long long n,
                          unsigned long long* bad);
double lex_sentinel_host();

// k_assembly.cu: Q1 assembly on the device (what: 0 mass, 1 Poisson, 2 SUPG
// convection-diffusion (eps), 3 partial-observation mass (obs = box, host
// array of 4)) into 9 coefficient arrays; transpose9; out = 1*a + 1*b.
void launch_assemble9(cudaStream_t s, int what, int level, double eps, const double* obs,
                      double* coef);
void launch_transpose9(cudaStream_t s, int nx, const double* in, double* out);
void launch_add9(cudaStream_t s, long long m, const double* a, const double* b, double* out);

// Cluster-resident bottom (k_mg_cluster.cu): levels <= 7 in one 16-CTA
// thread-block cluster with distributed shared memory. ops[0] is the top
// level handled (level 7 or 6).
using ClusterArgs = BottomArgs;
constexpr int kClusterTopLevel = 7;
bool cluster_bottom_supported();
bool cluster_top8_supported(); // the level-8 (constant stencil + diagonal) variant fits this device
// tuning aid: enable %globaltimer phase probes; read the last launch's stamps
void cluster_probes(int enable, unsigned long long* out64);
void lex_probes(int enable, unsigned long long* out512); // lexicographic sweep stamps
void launch_bottom_cluster(cudaStream_t s, const ClusterArgs& a, const double* b, double* x,
                           int cycles, int pre, int post, bool check, double* state, int* flags);
// Chained level-8 solves in ONE launch (the heat time-block substitution,
// timedep.cpp:268-311): batch elements first, first + dbt, ... (nblk of them;
// `a`, r and x address the first). Element j > 0 solves A_j x_j = r_j + M x_{j-1}
// with M the constant 9-point stencil mc (k_rhs_plus_mass's arithmetic), x_{j-1}
// taken from shared memory. ns = nodes per element (stride of r, x and the
// fine diagonal; coarse operators, LU and dense operator are batch-contiguous).
struct ChainArgs {
    int nblk;
    int dbt;
    long long ns;
    double mc[9];
};
void launch_cluster_chain(cudaStream_t s, const ClusterArgs& a, const double* r, double* x,
                          const ChainArgs& ch, int cycles, int pre, int post, bool check,
                          double* state, int* flags);
extern std::atomic<int> g_heat_chain; // 1: a heat substitution direction is one chained cluster launch
// Dense operator of the V-cycle below level 5 (levels 4, 3 and the level-2 LU)
// for the cluster kernel: a.ops[0] = level 4, a.ops[1] = level 3 of batch
// element 0 (elements are 9 n_k apart), lu/perm of element 0; out: batch x 225 x 225.
constexpr int kCoarseOpN = 225;
void launch_coarse_op(cudaStream_t s, const BottomArgs& a, int batch, int pre, int post, double* out);

} // namespace ocb

namespace ocb {

// ------------------------------------------------------------- problem ops
// Device view of the saddle-system blocks (reference ipm.cpp:347-374 for the
// steady model, timedep.cpp:18-133 for the space-time heat model).
struct ProbDev {
    int nx;             // spatial interior nodes per side
    long long ns;       // spatial nodes per block (nx*nx)
    int nt;             // time blocks (1 for steady problems)
    long long ny;       // ns * nt
    int heat;           // 1 = space-time heat model
    int has_sb;         // state box present (theta_y, lam_y used)
    Op9 L;              // constraint operator K (steady): Poisson or SUPG convdiff
    Op9 LT;             // K^T (steady)
    Op9 M;              // consistent mass (constant stencil)
    Op9 Mobs;           // observation mass (M or the partial mass)
    Op9 Mtl;            // heat: M + tau L (constant stencil)
    double alpha, beta, tau;
    const double* qw;   // heat: quadrature weight per time block (device)
};

// out = A x for the reduced saddle operator (make_saddle_operator,
// ipm.cpp:237-268); if part != nullptr, instead accumulate |b - A x|^2 block
// partials (true residual, krylov.cpp:23-34) and optionally still write out.
void launch_kkt(cudaStream_t s, const ProbDev& P, const double* ty, const double* tw,
                const double* tv, const double* x, double* out, const double* b, double* part);

// Chebyshev semi-iteration on s_k*M + diag(e) per block (chebyshev.cpp:49-75).
// e may be null (zero extra diagonal). Writes the result to out[0..ny).
struct ChebWork {
    double* g;
    double* r0;
    double* r1;
    double* r2;
};
void launch_chebyshev(cudaStream_t s, const ProbDev& P, const double* b, const double* e,
                      int steps, const ChebWork& w, double* out);
extern std::atomic<int> g_cheb_block; // 1: up to 5 Chebyshev steps per launch (temporal blocking)
extern std::atomic<int> g_kkt_tiled;  // 1: steady KKT apply from shared-memory halo tiles
extern std::atomic<int> g_heat_fork;  // 1: heat P_D's time-block substitution on the high-priority side stream
extern std::atomic<long long> g_tuning_gen; // bumped by every oc_set_tuning (invalidates graphs)
extern std::atomic<int> g_fuse_norm;  // 1: a V-cycle's last sweep launch runs the divergence check
extern std::atomic<int> g_fuse_restrict; // 1: a level's last pre-smoothing launch restricts the residual

// 2x2 control block inverse (precond.cpp:37-53, 148-157; heat timedep.cpp:383-393)
void launch_control_2x2(cudaStream_t s, const ProbDev& P, const double* tw, const double* tv,
                        const double* rw, const double* rv, double* vw, double* vv,
                        int* flags);
// P_T coupling row: steady t = L vy - M vw + M vv - rp (precond.cpp:223-227);
// heat t = Ldt vy - tau M (vw - vv) - rp (timedep.cpp:411-418)
void launch_coupling(cudaStream_t s, const ProbDev& P, const double* vy, const double* vw,
                     const double* vv, const double* rp, double* t);
// Schur middle: steady t2 = M_obs t1 + theta_y t1 (precond.cpp:133-134);
// heat u_k = tau w_k M t_k + theta_y t_k (timedep.cpp:289-296). ty may be null.
void launch_schur_middle(cudaStream_t s, const ProbDev& P, const double* ty, const double* t1,
                         double* t2);
// matching diagonals: steady bracket = d^2 s/(alpha d s + 1) (precond.cpp:55-72),
// mhat = sqrt(bracket) sqrt(d + theta_y) (precond.cpp:74-84); heat time_m_hat
// (timedep.cpp:215-243). Either output may be null; ty may be null (zero).
void launch_mhat(cudaStream_t s, const ProbDev& P, const double* ty, const double* tw,
                 const double* tv, double* mhat, double* bracket, int* flags);
// out[i] = a[i] + b[i] over n (9-point coefficient sums, e.g. L^T + M_obs)
void launch_add(cudaStream_t s, const double* a, const double* b, double* out, long long n);
// P_Pi pieces (precond.cpp:287-308):
// rhs1 = M (v2w - v2v) + rp
void launch_ppi_rhs1(cudaStream_t s, const ProbDev& P, const double* vw, const double* vv,
                     const double* rp, double* rhs1);
// t = M_obs v1 + (theta_y v1 - ry)
void launch_ppi_t(cudaStream_t s, const ProbDev& P, const double* ty, const double* v1,
                  const double* ry, double* t);
// y = A x for a single 9-point operator (steady field)
void launch_op_apply(cudaStream_t s, const Op9& A, const double* x, double* y);
// heat: out_k = M x_{k-1} added (forward) or M x_{k+1} (backward) into rhs_k:
// rhs = r_k + M x_nb  (timedep.cpp:277-286, 300-309)
void launch_rhs_plus_mass(cudaStream_t s, const ProbDev& P, const double* r, const double* xnb,
                          double* rhs);

// --------------------------------------------------------------- vectors
void launch_dot_partials(cudaStream_t s, const double* x, const double* y, long long n,
                         double* part);
// dst = op(sum partials): mode 0 sum, 1 sqrt(sum)
void launch_finalize(cudaStream_t s, const double* part, double* dst, int mode);
void launch_copy(cudaStream_t s, const double* x, double* y, long long n);
void launch_fill(cudaStream_t s, double* x, double v, long long n);
// y = x * (1/ *den)     (scaled(1.0/den, x))
void launch_scale_inv(cudaStream_t s, const double* x, const double* den, double* y, long long n,
                      const int* stop);
// w += (-(*h)) * v      (axpy(-h, v, w))
void launch_axpy_neg(cudaStream_t s, const double* h, const double* v, double* w, long long n);
// x = sum_i y[i] * Z_i with Z_i = Ztab[i] (device pointer table), the GMRES
// iterate rebuild (krylov.cpp:196-197)
// If xbase != nullptr: x = xbase + sum (restarted GMRES).
void launch_combine(cudaStream_t s, const double* const* Ztab, const double* y, int m, double* x,
                    long long n, const double* xbase = nullptr);

// ----------------------------------------------------------------- GMRES
// Device state of one GMRES solve (krylov.cpp:133-212); H column-major
// (ld = maxit+1), cs/sn/g rotations, y the current LS solution.
struct GmresDev {
    double* H;      // (maxit+1) x maxit
    double* cs;
    double* sn;
    double* g;      // maxit+1
    double* y;      // maxit
    double* scal;   // [0] bnorm, [1] hnext, [2] relres, [3] h_i scratch
    int* stop;      // 0 running, 1 zero pivot
    int ld;
};
// h_i = <w, V_i> from partials, stored at H(i, j); then w -= h_i V_i
// MGS step i + the next dot: w -= h_ij v_i (h_ij from part_in), part_out = partials
// of <w, vnext> (vnext == w: ||w||^2), bit-identical to dot_partials after mgs_step
// the first inner product of the orthogonalisation, on the kMgsBlocks grid
void launch_dot_partials_mgs(cudaStream_t s, const double* x, const double* y, long long n,
                             double* part);
void launch_mgs_dot(cudaStream_t s, const double* part_in, const GmresDev& G, int i, int j,
                    const double* vi, double* w, const double* vnext, double* part_out, long long n);
void launch_mgs_step(cudaStream_t s, const double* part, const GmresDev& G, int i, int j,
                     const double* vi, double* w, long long n);
// the whole MGS of column j (the dot + j+1 mgs_dot launches above, same bits) in
// one cooperative launch with w in shared memory; false = not applicable here
// (n too large, not a 148-SM device). Step j's partials land in (j & 1) ? pa : pb.
bool launch_mgs_persistent(cudaStream_t s, const double* const* V, double* w, const GmresDev& G,
                           int j, double* pa, double* pb, unsigned* bar, long long n);
// hnext from partials -> H(j+1, j), Givens update and back substitution for y (one thread)
void launch_gmres_givens(cudaStream_t s, const double* part, const GmresDev& G, int j);
// scal[2] = sqrt(sum part) / bnorm
// (status != nullptr: also status[0] = flags[0], status[1] = stop[0], as doubles)
void launch_gmres_status(cudaStream_t s, const GmresDev& G, int j, const int* flags, double* est,
                         double* status);
extern std::atomic<int> g_gmres_lazy_residual; // 1: true residual only once the carried estimate nears the tolerance
void launch_relres(cudaStream_t s, const double* part, const double* bnorm, double* dst,
                   const int* flags = nullptr, const int* stop = nullptr, double* status = nullptr);

// ----------------------------------------------------------------- MINRES
// scalar state (krylov.cpp:37-131): see k_vec.cu for the slot layout
void launch_minres_setup(cudaStream_t s, const double* part, double* sc);
void launch_minres_delta(cudaStream_t s, const double* part, double* sc);
void launch_minres_vnext(cudaStream_t s, const double* az, const double* v, const double* vprev,
                         double* vnext, const double* sc, int first, long long n);
void launch_minres_gamma(cudaStream_t s, const double* part, double* sc, int* stop);
void launch_minres_update(cudaStream_t s, const double* z, const double* wprev, const double* w,
                          double* wnext, double* x, const double* sc, const int* stop,
                          long long n);
void launch_minres_rotate(cudaStream_t s, double* sc, const int* stop);


// ------------------------------------------------------------------- IPM
// Device state of the interior point iteration (ipm.hpp:36-42) and the
// problem vectors of the model (ipm.hpp:83-88).
struct IpmDev {
    double *y, *z, *p, *lya, *lyb, *lza, *lzb;
    const double *yd, *f, *za, *zb, *ya, *yb, *ld;
    double *ty, *tw, *tv;
    double *dy, *dz, *dp, *dlya, *dlyb, *dlza, *dlzb;
};
// build_theta (ipm.cpp:32-61)
void launch_theta(cudaStream_t s, const ProbDev& P, const IpmDev& S, int* flags);
// newton_rhs (ipm.cpp:112-143) into rhs = [r1 | r2 | r3]
void launch_newton_rhs(cudaStream_t s, const ProbDev& P, const IpmDev& S, double mu, double* rhs);
// recover_multiplier_steps + ratio partials (ipm.cpp:145-210); part: 2*kRedBlocks mins
void launch_recover_ratios(cudaStream_t s, const ProbDev& P, const IpmDev& S, double mu,
                           double* part);
// alpha_P, alpha_D = min(1, alpha0 * ratio) -> steps[0..1]
void launch_step_lengths(cudaStream_t s, const double* part, double alpha0, double* steps);
// state update + interiority checks (ipm.cpp:305-319)
void launch_ipm_update(cudaStream_t s, const ProbDev& P, const IpmDev& S, const double* steps,
                       int* flags);
// ipm_residuals squared sums (ipm.cpp:63-110): part 3*kRedBlocks -> norms[0..2] (RMS)
void launch_ipm_residuals(cudaStream_t s, const ProbDev& P, const IpmDev& S, double mu,
                          double* part, double* norms);
// objective (qp.cpp:112-121 / heat closures) and sparsity of u = w - v
// out: [0] J, [1] count |u|<thr, [2] l1
void launch_objective(cudaStream_t s, const ProbDev& P, const IpmDev& S, double* part,
                      double* out);
// initial_point (ipm.cpp:212-235)
void launch_initial_point(cudaStream_t s, const ProbDev& P, const IpmDev& S);
// problem setup on the device (build_qp qp.cpp:123-174 vectors)
void launch_split_bounds(cudaStream_t s, long long ns, int nt, const double* ua, const double* ub,
                         double* za, double* zb, int* flags);
void launch_check_state_bounds(cudaStream_t s, long long n, const double* ya, const double* yb,
                               int* flags);
void launch_lumped(cudaStream_t s, int nx, const Op9& M, double* ld);
void launch_replicate(cudaStream_t s, long long ns, int nt, double scale, const double* in,
                      double* out);
// u = w - v
void launch_recover_control(cudaStream_t s, long long ny, const double* z, double* u);

} // namespace ocb
