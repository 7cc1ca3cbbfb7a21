// Host orchestration of the device-resident IPM Newton solve.
//
// Everything here only enqueues kernels on the context stream; the host reads
// back a handful of scalars once per Krylov iteration (convergence test) and
// once per IPM iteration (residual norms, error flags).
#pragma once

#include "../../include/optcon_b200.h"
#include "kernels.hpp"

#include <map>
#include <memory>
#include <tuple>
#include <stdexcept>
#include <string>
#include <vector>

namespace ocb {

struct InvalidArgument : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};
struct RuntimeError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct CudaFailure : std::runtime_error {
    using std::runtime_error::runtime_error;
};

void cuda_check(cudaError_t e, const char* what);

// Device memory comes from the stream-ordered pool allocator on the per-thread
// stream: cudaFree would synchronise the whole device and serialise concurrent
// solves (one context per host thread); pooled blocks are also reused across
// problems. Owners synchronise their solver stream before releasing memory.
void* pool_alloc(size_t bytes);
void pool_free(void* p);

template <typename T>
class DevArray {
public:
    DevArray() = default;
    explicit DevArray(size_t n) { resize(n); }
    ~DevArray() { release(); }
    DevArray(const DevArray&) = delete;
    DevArray& operator=(const DevArray&) = delete;
    DevArray(DevArray&& o) noexcept : p_(o.p_), n_(o.n_) { o.p_ = nullptr; o.n_ = 0; }
    DevArray& operator=(DevArray&& o) noexcept
    {
        if (this != &o) {
            release();
            p_ = o.p_; n_ = o.n_;
            o.p_ = nullptr; o.n_ = 0;
        }
        return *this;
    }
    void resize(size_t n)
    {
        if (n == n_) return;
        release();
        if (n) p_ = static_cast<T*>(pool_alloc(n * sizeof(T)));
        n_ = n;
    }
    void release()
    {
        if (p_) pool_free(p_);
        p_ = nullptr;
        n_ = 0;
    }
    T* get() const { return p_; }
    size_t size() const { return n_; }
    explicit operator bool() const { return p_ != nullptr; }

private:
    T* p_ = nullptr;
    size_t n_ = 0;
};
using DVec = DevArray<double>;

// Per-launch CUDA-event spans on the solver stream for the bench's in-situ
// kernel timing (fine-level smoothing sweeps, KKT applies, P applies).
// kProfBlock: one heat time-block multigrid solve (the level-8 cluster launch)
enum ProfCat { kProfSweep = 0, kProfKkt = 1, kProfPrec = 2, kProfBlock = 3, kProfCats = 4 };
struct Profiler {
    bool on = false;
    struct Span {
        cudaEvent_t a = nullptr, b = nullptr;
        int cat = 0;
    };
    std::vector<Span> spans;
    size_t used = 0;
    int begin(cudaStream_t s, int cat);
    void end(cudaStream_t s, int idx);
    // sum elapsed per category (syncs), then reset
    void read(double* ms, long long* counts);
    ~Profiler();
};

struct Ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    // high-priority side stream: the heat time-block substitution of a P_D
    // apply runs on it, forked from / joined to `stream` by two events, while
    // the Chebyshev and 2x2 blocks run on `stream`
    cudaStream_t side = nullptr;
    cudaStream_t lexs[kLexPipe - 1] = {}; // sweeps 2.. of a pipelined lexicographic batch
    cudaEvent_t lex_fork = nullptr, lex_ev[kLexPipe - 1] = {};
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    cudaEvent_t user_ev[8] = {};
    double* hscal = nullptr; // pinned host mirror (64 doubles)
    int* hflags = nullptr;   // pinned host mirror (8 ints)
    Profiler prof;
    // Instantiated preconditioner graphs released by closed problems, kept for
    // the next problem on this context: a new capture of the same apply shape
    // is patched into one with cudaGraphExecUpdate instead of instantiated.
    struct SpareGraph {
        long long launches;
        cudaGraphExec_t exec;
    };
    std::vector<SpareGraph> spare_graphs;
    static constexpr size_t kMaxSpareGraphs = 64;
    explicit Ctx(int dev);
    ~Ctx();
    void sync();
};

// RAII span: no-op unless profiling is on
struct ProfScope {
    Ctx& c;
    int idx;
    ProfScope(Ctx& cx, int cat)
        : c(cx), idx((cx.prof.on && cat < kProfCats) ? cx.prof.begin(cx.stream, cat) : -1)
    {
    }
    ~ProfScope()
    {
        if (idx >= 0) c.prof.end(c.stream, idx);
    }
};

// Copy between host/device pointers of unknown kind (cudaMemcpyDefault).
void copy_any(Ctx& c, void* dst, const void* src, size_t bytes);
bool is_device_ptr(const void* p);

struct MgParams {
    int cycles = 3, pre = 5, post = 5;
};

// Geometric multigrid hierarchy (MgHierarchy, multigrid.hpp:43-64) for one
// operator, or for `batch` operators of the same level (heat time blocks).
class Hierarchy {
public:
    // smoother: OC_SMOOTHER_COLOR4 or OC_SMOOTHER_LEX (reference order, in place)
    void allocate(int level, int batch = 1, int smoother = OC_SMOOTHER_COLOR4);
    // Galerkin coarse operators R A P of the fine operator (per batch block the
    // fine coef/diag pointers advance by fine_coef_stride / fine_diag_stride).
    void build(Ctx& c, const Op9& fine, long long fine_coef_stride = 0,
               long long fine_diag_stride = 0);
    // Rediscretised coarse operators: base[k] (k = 1..K, 9 arrays each) plus
    // the Galerkin-coarsened remainder fine - base(level) (multigrid.cpp:86-101).
    void build_rediscretized(Ctx& c, const Op9& fine, const std::vector<const double*>& base);
    // solve: `cycles` V-cycles from x = 0 with the divergence check.
    void solve(Ctx& c, const double* b, double* x, const MgParams& p, int bt, int* flags);
    // the heat substitution in one chained cluster launch: batch elements
    // first, first + step, ... (count of them), element j solving
    // A_j x_j = r_j + M x_{j-1}; r and x are whole space-time vectors.
    // Returns false (nothing launched) when this hierarchy cannot chain.
    bool can_chain(const MgParams& p, const Op9& M) const;
    bool solve_chain(Ctx& c, const double* r, double* x, const MgParams& p, int first, int step,
                     int count, const Op9& M, int* flags);
    // one smoothing sweep on the fine level (in place through the scratch buffer)
    void smooth(Ctx& c, const double* b, double* x, bool forward, int bt);
    // cluster bottom: (re)compute the dense levels <= 4 cycle operator for these
    // sweep counts if stale (build() invalidates it); enqueued on c's stream
    void ensure_coarse_op(Ctx& c, int pre, int post);
    const double* coarse_op() const { return cluster_ ? cop_.get() : nullptr; }
    int depth() const { return K_; }
    bool built() const { return built_; }
    int level() const { return level_; }
    int smoother() const { return smoother_; }
    // bumped whenever allocate() (re)allocates device buffers: captured graphs
    // that bake in this hierarchy's pointers are then stale
    long long generation() const { return gen_; }
    Op9 level_op(int k, int bt) const;
    long long level_n(int k) const { return (long long)nx_[k] * nx_[k]; }

private:
    void vcycle(Ctx& c, int k, const double* b, double* xout, bool zero_in, const MgParams& p,
                int bt, int* flags, bool* fused_norm = nullptr);
    BottomArgs bottom_args(int kfrom, int bt) const;
    void build_inv(Ctx& c);
    void build_split(Ctx& c);
    const double* inv_at(int k, int bt) const { return inv_[k].get() + (size_t)bt * level_n(k); }
    const double* dfull_at(int k, int bt) const { return dfull_[k].get() + (size_t)bt * level_n(k); }

    int level_ = 0, K_ = 0, kb_ = 0, batch_ = 1, smoother_ = OC_SMOOTHER_COLOR4;
    bool lex_ = false;     // lexicographic smoother: in-place wavefront sweeps, single-CTA bottom
    long long gen_ = 0;
    DVec mbox_;            // wavefront hand-off mailboxes (lex): kLexPipe sets of ceil(nx/32) * nx sentinels
    DevArray<int> prog_;   // per-band progress counters of a pipelined batch (kLexPipe x (bands + 1))
    // `count` lexicographic sweeps of level k (pipelined when enabled)
    void lex_sweeps(Ctx& c, const Op9& A, const double* b, int k, int bt, double* x, bool forward,
                    int count, int* flags);
    bool cluster_ = false;  // bottom levels run in the 16-CTA cluster kernel
    std::vector<int> nx_;
    Op9 fine_{};
    long long fine_coef_stride_ = 0, fine_diag_stride_ = 0;
    std::vector<DVec> coef_;        // [k] 9*n_k*batch, k >= 1
    std::vector<DVec> rem_;         // rediscretised remainder chain, k >= 1 (batch 1)
    DVec remfine_;                  // fine remainder fine - base(level), 9 arrays
    std::vector<DVec> xa_, xb_, b_; // per level work (k >= 1); xb_[0] fine scratch
    std::vector<DVec> inv_;         // 1/diag per tiled level (k < kb_), batch-strided
    std::vector<DVec> dfull_;       // lexicographic mode: the diagonal values themselves
    DVec lu_;
    DevArray<int> perm_;
    std::vector<DVec> split_;       // [k] colour-split off-diagonal records of variable tiled levels >= 511^2 (batch 1)
    DVec cop_;                      // cluster: batch x 225 x 225 dense levels <= 4 cycle operator
    int cop_pre_ = -1, cop_post_ = -1; // sweep counts cop_ was computed for (-1: stale)
    DVec part_, state_;
    DevArray<unsigned> cnt_; // last-block counter of the fused divergence check
    bool built_ = false;
};

class Problem {
public:
    Problem(Ctx& c, const oc_problem_desc& d);
    ~Problem(); // synchronises before members return memory to the pool
    oc_problem_info info() const;

    // preconditioner setup from Theta already in ty_/tw_/tv_ (device)
    void setup_precond(int kind, const oc_ipm_params& p);
    void precond_apply(int kind, const double* r, double* out);
    void precond_apply_direct(int kind, const double* r, double* out);
    void schur_apply(const double* r, double* out);
    void kkt(const double* x, double* out);
    void set_theta(const double* ty, const double* tw, const double* tv);

    oc_solve_report newton_solve(const oc_ipm_params& p, const double* rhs, double* x);
    void ipm_solve(const oc_ipm_params& p, oc_ipm_result* r);
    void ipm_pieces(const double* y, const double* z, const double* pv, const double* lya,
                    const double* lyb, const double* lza, const double* lzb, double mu_state,
                    double mu_rhs, double* ty, double* tw, double* tv, double* r1, double* r2,
                    double* r3, double* norms3);
    double objective(const double* y, const double* z);
    void time_applies(int kind, int reps, double* kkt_ms, double* prec_ms);

    Ctx& ctx;
    ProbDev P{};
    IpmDev S{};

private:
    void check_flags(bool sync_now = true);
    void upload(DVec& dst, const double* src, size_t n);
    oc_solve_report gmres(const oc_ipm_params& p, int kind, const double* b, double* x);
    oc_solve_report minres(const oc_ipm_params& p, int kind, const double* b, double* x);
    void time_schur(const double* r, double* out);
    double read_scalar(const double* dptr);
    void ensure_krylov(size_t count);

    int level_ = 0, nx_ = 0, nt_ = 1;
    long long ns_ = 0, ny_ = 0;
    long long h2d_bytes_ = 0;
    bool heat_ = false, has_sb_ = false, partial_obs_ = false, convdiff_ = false;
    double eps_ = 0.0;
    MgParams mg_{};
    int cheb_steps_ = 20;

    // operators and problem data
    DVec Lc_, LTc_, Mobsc_, LTpMobs_;
    std::vector<DVec> base_, baseT_;
    DVec yd_, f_, za_, zb_, ya_, yb_, ld_, qw_;
    // state and directions
    DVec y_, z_, p_, lya_, lyb_, lza_, lzb_;
    DVec dlya_, dlyb_, dlza_, dlzb_;
    DVec ty_, tw_, tv_;
    DVec rhs_, sol_;
    // preconditioner
    DVec mhat_, bracket_;
    DVec cg_, c0_, c1_, c2_;
    DVec t_, t2_, t3_, tf_, rblk_;
    Hierarchy HF_, HFT_, HL_, Hleft_, Hright_, Hheat_;
    bool HL_built_ = false;
    int smoother_ = OC_SMOOTHER_COLOR4;
    int setup_kind_ = -1;
    // CUDA graphs of the preconditioner apply, keyed by (kind, r, out, MG and
    // Chebyshev parameters): captured on the second use of a key, replayed
    // afterwards (one launch instead of ~200). Device pointers baked into the
    // graphs are stable across Newton steps; any hierarchy reallocation (see
    // Hierarchy::generation) drops them.
    struct GraphEntry {
        cudaGraphExec_t exec = nullptr;
        int uses = 0;
        long long launches = 0;
    };
    using GraphKey = std::tuple<int, const void*, const void*, int, int, int, int, int, int>;
    std::map<GraphKey, GraphEntry> graphs_;
    long long graph_gen_ = -1;
    bool graphs_enabled_ = true;
    void drop_graphs();
    long long hierarchy_generation() const;
    // Krylov
    std::vector<DVec> V_, Z_;
    DevArray<const double*> Ztab_, Vtab_; // device tables of the Z / V basis pointers
    DevArray<unsigned> gbar_;             // grid barrier of the persistent MGS launch
    DVec kw_, kx2_, kvec_[8];
    DVec H_, cs_, sn_, g_, yls_;
    // scalars
    DVec part_, scal_;
    DevArray<int> flags_, stop_;
};

} // namespace ocb
