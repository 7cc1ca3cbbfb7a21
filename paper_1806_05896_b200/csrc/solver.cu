// Host orchestration of the device-resident IPM Newton solve (see solver.hpp).
//
// Reference call structure reproduced here:
//   ipm_solve                      ipm.cpp:270-341
//   make_steady_model/newton_solve ipm.cpp:388-470
//   make_spacetime_model           timedep.cpp:313-441
//   Block11Approx/SchurApprox/...  precond.cpp:110-308
//   MgHierarchy build/solve        multigrid.cpp:75-157
//   minres / gmres                 krylov.cpp:37-212
#include "solver.hpp"

#include <nvtx3/nvToolsExt.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>

#include "assembly.hpp"

#include <algorithm>
#include <cmath>
#include <atomic>
#include <mutex>
#include <cstdlib>
#include <cstring>

namespace ocb {

// NVTX ranges around the solver phases (ipm_solve, each Newton step's
// preconditioner setup and Krylov solve): visible in Nsight timelines,
// a no-op without an attached tool
struct Nvtx {
    explicit Nvtx(const char* name) { nvtxRangePushA(name); }
    ~Nvtx() { nvtxRangePop(); }
    Nvtx(const Nvtx&) = delete;
    Nvtx& operator=(const Nvtx&) = delete;
};

void cuda_check(cudaError_t e, const char* what)
{
    if (e != cudaSuccess) throw CudaFailure(std::string(what) + ": " + cudaGetErrorString(e));
}

static void launch_check(const char* what) { cuda_check(cudaGetLastError(), what); }

void* pool_alloc(size_t bytes)
{
    static std::once_flag once;
    std::call_once(once, [] {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            unsigned long long keep = ~0ull; // keep freed blocks pooled
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        }
    });
    void* p = nullptr;
    cuda_check(cudaMallocAsync(&p, bytes, cudaStreamPerThread), "cudaMallocAsync");
    // the allocation is ordered on the per-thread stream; make it usable from
    // the solver stream without a device-wide synchronisation
    cuda_check(cudaStreamSynchronize(cudaStreamPerThread), "cudaStreamSynchronize");
    return p;
}

void pool_free(void* p)
{
    cudaFreeAsync(p, cudaStreamPerThread);
}

static std::atomic<long long> g_launches{0};
static thread_local long long t_launches = 0; // this host thread's launches (graph capture)
void note_launch()
{
    g_launches.fetch_add(1, std::memory_order_relaxed);
    ++t_launches;
}
static std::atomic<int> g_contexts{0};
int active_contexts() { return g_contexts.load(std::memory_order_relaxed); }
void add_launches(long long k) { g_launches.fetch_add(k, std::memory_order_relaxed); }
long long launch_count() { return g_launches.load(std::memory_order_relaxed); }

int Profiler::begin(cudaStream_t s, int cat)
{
    if (used == spans.size()) {
        Span sp;
        cuda_check(cudaEventCreate(&sp.a), "cudaEventCreate");
        cuda_check(cudaEventCreate(&sp.b), "cudaEventCreate");
        spans.push_back(sp);
    }
    spans[used].cat = cat;
    cudaEventRecord(spans[used].a, s);
    return (int)used++;
}

void Profiler::end(cudaStream_t s, int idx) { cudaEventRecord(spans[idx].b, s); }

void Profiler::read(double* ms, long long* counts)
{
    for (int k = 0; k < kProfCats; ++k) {
        ms[k] = 0.0;
        counts[k] = 0;
    }
    for (size_t i = 0; i < used; ++i) {
        cuda_check(cudaEventSynchronize(spans[i].b), "cudaEventSynchronize");
        float t = 0.f;
        cuda_check(cudaEventElapsedTime(&t, spans[i].a, spans[i].b), "cudaEventElapsedTime");
        ms[spans[i].cat] += t;
        counts[spans[i].cat] += 1;
    }
    used = 0;
}

Profiler::~Profiler()
{
    for (auto& s : spans) {
        cudaEventDestroy(s.a);
        cudaEventDestroy(s.b);
    }
}

Ctx::Ctx(int dev) : device(dev)
{
    int count = 0;
    cuda_check(cudaGetDeviceCount(&count), "cudaGetDeviceCount");
    if (dev < 0 || dev >= count) throw CudaFailure("oc_create: no such CUDA device");
    cuda_check(cudaSetDevice(dev), "cudaSetDevice");
    cuda_check(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking), "cudaStreamCreate");
    int lo = 0, hi = 0;
    cuda_check(cudaDeviceGetStreamPriorityRange(&lo, &hi), "cudaDeviceGetStreamPriorityRange");
    cuda_check(cudaStreamCreateWithPriority(&side, cudaStreamNonBlocking, hi), "cudaStreamCreate");
    cuda_check(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming), "cudaEventCreate");
    cuda_check(cudaEventCreateWithFlags(&lex_fork, cudaEventDisableTiming), "cudaEventCreate");
    for (int q = 0; q < kLexPipe - 1; ++q) {
        cuda_check(cudaStreamCreateWithFlags(&lexs[q], cudaStreamNonBlocking), "cudaStreamCreate");
        cuda_check(cudaEventCreateWithFlags(&lex_ev[q], cudaEventDisableTiming), "cudaEventCreate");
    }
    cuda_check(cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming), "cudaEventCreate");
    cuda_check(cudaEventCreate(&ev0), "cudaEventCreate");
    cuda_check(cudaEventCreate(&ev1), "cudaEventCreate");
    for (auto& e : user_ev) cuda_check(cudaEventCreate(&e), "cudaEventCreate");
    cuda_check(cudaMallocHost(&hscal, 64 * sizeof(double)), "cudaMallocHost");
    cuda_check(cudaMallocHost(&hflags, 8 * sizeof(int)), "cudaMallocHost");
    g_contexts.fetch_add(1, std::memory_order_relaxed);
}

Ctx::~Ctx()
{
    g_contexts.fetch_sub(1, std::memory_order_relaxed);
    if (stream) cudaStreamSynchronize(stream);
    if (hscal) cudaFreeHost(hscal);
    if (hflags) cudaFreeHost(hflags);
    if (ev0) cudaEventDestroy(ev0);
    if (ev1) cudaEventDestroy(ev1);
    for (auto& e : user_ev)
        if (e) cudaEventDestroy(e);
    for (auto& g : spare_graphs) cudaGraphExecDestroy(g.exec);
    if (side) {
        cudaStreamSynchronize(side);
        cudaStreamDestroy(side);
    }
    for (int q = 0; q < kLexPipe - 1; ++q) {
        if (lexs[q]) {
            cudaStreamSynchronize(lexs[q]);
            cudaStreamDestroy(lexs[q]);
        }
        if (lex_ev[q]) cudaEventDestroy(lex_ev[q]);
    }
    if (lex_fork) cudaEventDestroy(lex_fork);
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
    if (stream) cudaStreamDestroy(stream);
}

void Ctx::sync() { cuda_check(cudaStreamSynchronize(stream), "cudaStreamSynchronize"); }

bool is_device_ptr(const void* p)
{
    if (!p) return false;
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

void copy_any(Ctx& c, void* dst, const void* src, size_t bytes)
{
    if (!bytes) return;
    cuda_check(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, c.stream), "cudaMemcpyAsync");
}

// =================================================================== Hierarchy
void Hierarchy::allocate(int level, int batch, int smoother)
{
    if (level < 3) throw InvalidArgument("MgHierarchy: fine level must be >= 3");
    if (smoother != OC_SMOOTHER_COLOR4 && smoother != OC_SMOOTHER_LEX)
        throw InvalidArgument("MgHierarchy: unknown smoother");
    if (built_ && level == level_ && batch == batch_ && smoother == smoother_) return;
    ++gen_;
    level_ = level;
    batch_ = batch;
    smoother_ = smoother;
    lex_ = smoother == OC_SMOOTHER_LEX;
    K_ = level - 2;
    nx_.assign(K_ + 1, 0);
    for (int k = 0; k <= K_; ++k) nx_[k] = (1 << (level - k)) - 1;
    // levels <= 7 run in the 16-CTA cluster kernel when the top of that range
    // is a slab level (>= 6); otherwise levels <= 6 in the single-CTA kernel
    // (the cluster kernel smooths with 4 colours; the lexicographic mode keeps
    // levels <= 6 in the single-CTA kernel and sweeps the others as wavefronts)
    cluster_ = !lex_ && g_cluster_bottom && level >= 6 && cluster_bottom_supported();
    // (lexicographic mode: levels 6 and 5 as wavefront bands of k_gs_lex,
    // faster than the single CTA's two warps streaming their coefficients;
    // C3 P_Pi apply 101 -> 92 ms)
    const int top = cluster_ ? kClusterTopLevel : (lex_ ? g_lex_bottom_top.load() : kBottomTopLevel);
    kb_ = 0;
    while (level - kb_ > top) ++kb_;
    coef_.clear();
    coef_.resize(K_ + 1);
    xa_.clear();
    xb_.clear();
    b_.clear();
    xa_.resize(K_ + 1);
    xb_.resize(K_ + 1);
    b_.resize(K_ + 1);
    for (int k = 1; k <= K_; ++k) {
        const size_t n = (size_t)level_n(k);
        coef_[k].resize(9 * n * batch);
        xa_[k].resize(n);
        xb_[k].resize(n);
        b_[k].resize(n);
    }
    xb_[0].resize((size_t)level_n(0));
    inv_.clear();
    inv_.resize(K_ + 1);
    dfull_.clear();
    dfull_.resize(K_ + 1);
    for (int k = 0; k < kb_; ++k) {
        inv_[k].resize((size_t)level_n(k) * batch);
        if (lex_) dfull_[k].resize((size_t)level_n(k) * batch);
    }
    if (lex_) {
        const int nx0 = nx_[0];
        mbox_.resize((size_t)kLexPipe * ((nx0 + 31) / 32) * nx0);
        prog_.resize((size_t)kLexPipe * ((nx0 + 31) / 32 + 1));
    } else {
        mbox_.release();
    }
    if (cluster_) cop_.resize((size_t)kCoarseOpN * kCoarseOpN * batch);
    else cop_.release();
    cop_pre_ = cop_post_ = -1;
    lu_.resize(81 * (size_t)batch);
    perm_.resize(9 * (size_t)batch);
    part_.resize(kNormBlocks);
    state_.resize(2);
    cnt_.resize(1);
    cuda_check(cudaMemsetAsync(cnt_.get(), 0, sizeof(unsigned), cudaStreamPerThread), "memset");
    cuda_check(cudaStreamSynchronize(cudaStreamPerThread), "cudaStreamSynchronize");
    built_ = true;
}

Op9 Hierarchy::level_op(int k, int bt) const
{
    if (k == 0) {
        Op9 a = fine_;
        if (a.coef) a.coef += bt * fine_coef_stride_;
        if (a.diag) a.diag += bt * fine_diag_stride_;
        a.csplit = bt == 0 && split_.size() > 0 && split_[0] ? split_[0].get() : nullptr;
        return a;
    }
    Op9 a{};
    a.nx = nx_[k];
    a.coef = coef_[k].get() + (size_t)bt * 9 * level_n(k);
    a.diag = nullptr;
    a.cscale = 1.0;
    a.csplit = bt == 0 && (size_t)k < split_.size() && split_[k] ? split_[k].get() : nullptr;
    return a;
}

void Hierarchy::build(Ctx& c, const Op9& fine, long long fcs, long long fds)
{
    // a constant-stencil level-8 operator (heat time blocks) runs its whole
    // solve in the cluster kernel (level 8 in 16-row bands)
    if (cluster_) {
        const int top = (level_ == 8 && !fine.coef && g_cluster_top8.load() && cluster_top8_supported())
                            ? 8
                            : kClusterTopLevel;
        kb_ = level_ > top ? level_ - top : 0;
    }
    fine_ = fine;
    fine_coef_stride_ = fcs;
    fine_diag_stride_ = fds;
    for (int k = 0; k < K_; ++k) {
        const Op9 f = level_op(k, 0);
        const long long cs = k == 0 ? fcs : 9 * level_n(k);
        const long long ds = k == 0 ? fds : 0;
        launch_rap(c.stream, f, coef_[k + 1].get(), nullptr, nullptr, batch_, cs, ds,
                   9 * level_n(k + 1));
    }
    launch_coarse_lu(c.stream, coef_[K_].get(), lu_.get(), perm_.get(), batch_);
    build_split(c);
    build_inv(c);
    launch_check("multigrid build");
}

void Hierarchy::ensure_coarse_op(Ctx& c, int pre, int post)
{
    if (!cluster_ || (pre == cop_pre_ && post == cop_post_)) return;
    BottomArgs a{};
    a.nlev = 3;
    for (int j = 0; j < 3; ++j) a.ops[j] = level_op(K_ - 2 + j, 0);
    a.lu = lu_.get();
    a.perm = perm_.get();
    launch_coarse_op(c.stream, a, batch_, pre, post, cop_.get());
    cop_pre_ = pre;
    cop_post_ = post;
}

void Hierarchy::build_split(Ctx& c)
{
    // tiled variable levels of >= 511^2 nodes sweep from colour-split copies
    // of their off-diagonals (one colour pass reads whole sectors); refreshed
    // at every build, as the coarse levels change with each Newton step
    const bool on = g_colour_split.load() && !lex_ && batch_ == 1;
    if (split_.size() != (size_t)K_ + 1) {
        split_.clear();
        split_.resize(K_ + 1);
    }
    for (int k = 0; k <= K_; ++k) {
        const double* src = k == 0 ? fine_.coef : coef_[k].get();
        const double* before = split_[k].get();
        if (!on || k >= kb_ || !src || nx_[k] < 500) {
            split_[k].release();
        } else {
            split_[k].resize((size_t)kSplitRecordWords * level_n(k));
            launch_colour_split(c.stream, nx_[k], src, k == 0 ? fine_.diag : nullptr, split_[k].get());
        }
        if (split_[k].get() != before) ++gen_; // captured graphs hold the old pointers
    }
}

void Hierarchy::build_inv(Ctx& c)
{
    cop_pre_ = cop_post_ = -1; // every (re)build ends here
    for (int k = 0; k < kb_; ++k) {
        const Op9 a = level_op(k, 0);
        const long long cs = k == 0 ? fine_coef_stride_ : 9 * level_n(k);
        const long long ds = k == 0 ? fine_diag_stride_ : 0;
        launch_inv_diag(c.stream, a, inv_[k].get(), batch_, cs, ds, lex_ ? dfull_[k].get() : nullptr);
    }
    if (lex_) launch_fill(c.stream, mbox_.get(), lex_sentinel_host(), (long long)mbox_.size());
}

void Hierarchy::build_rediscretized(Ctx& c, const Op9& fine, const std::vector<const double*>& base)
{
    if (batch_ != 1) throw InvalidArgument("rediscretised hierarchies are not batched");
    if (cluster_) kb_ = level_ > kClusterTopLevel ? level_ - kClusterTopLevel : 0;
    fine_ = fine;
    fine_coef_stride_ = fine_diag_stride_ = 0;
    if (rem_.size() != (size_t)K_ + 1) {
        rem_.clear();
        rem_.resize(K_ + 1);
        for (int k = 1; k <= K_; ++k) rem_[k].resize(9 * (size_t)level_n(k));
        remfine_.resize(9 * (size_t)level_n(0));
    }
    // remainder = A_f - base(level_f); coarse = base(l-1) + R remainder P
    launch_remainder9(c.stream, fine, base[0], remfine_.get());
    Op9 rem{};
    rem.nx = nx_[0];
    rem.coef = remfine_.get();
    rem.cscale = 1.0;
    for (int k = 0; k < K_; ++k) {
        launch_rap(c.stream, rem, coef_[k + 1].get(), base[k + 1], rem_[k + 1].get(), 1, 0, 0,
                   9 * level_n(k + 1));
        rem.nx = nx_[k + 1];
        rem.coef = rem_[k + 1].get();
    }
    launch_coarse_lu(c.stream, coef_[K_].get(), lu_.get(), perm_.get(), 1);
    build_split(c);
    build_inv(c);
    launch_check("multigrid build (rediscretised)");
}

BottomArgs Hierarchy::bottom_args(int kfrom, int bt) const
{
    BottomArgs a{};
    a.nlev = K_ - kfrom + 1;
    a.lex = lex_ ? 1 : 0;
    if (a.nlev > kBottomMaxLevels) throw RuntimeError("bottom solver: too many levels");
    for (int j = 0; j < a.nlev; ++j) a.ops[j] = level_op(kfrom + j, bt);
    a.lu = lu_.get() + 81 * (size_t)bt;
    a.perm = perm_.get() + 9 * (size_t)bt;
    a.cop = cluster_ ? cop_.get() + (size_t)kCoarseOpN * kCoarseOpN * bt : nullptr;
    return a;
}

void Hierarchy::lex_sweeps(Ctx& c, const Op9& A, const double* b, int k, int bt, double* x,
                           bool forward, int count, int* flags)
{
    const double* inv = inv_at(k, bt);
    const double* dfull = dfull_at(k, bt);
    const int nb0 = (nx_[0] + 31) / 32;
    const size_t mstride = (size_t)nb0 * nx_[0]; // one mailbox set
    const int pstride = nb0 + 1;
    if (!g_lex_pipeline.load() || count < 2) {
        for (int s = 0; s < count; ++s)
            launch_gs_lex(c.stream, A, b, inv, dfull, x, forward, mbox_.get(), flags);
        return;
    }
    // Sweep q+1 of a batch trails sweep q by a few chunks per band instead of
    // a whole sweep: every sweep is its own launch on its own stream (fork /
    // join by events, capturable), with its own mailbox set; the kernels pace
    // each other through per-band progress counters (k_mg_lex.cu).
    for (int done = 0; done < count; done += kLexPipe) {
        const int m = std::min(kLexPipe, count - done);
        cuda_check(cudaMemsetAsync(prog_.get(), 0, sizeof(int) * (size_t)m * pstride, c.stream), "memset");
        cuda_check(cudaEventRecord(c.lex_fork, c.stream), "cudaEventRecord");
        for (int q = 0; q < m; ++q) {
            cudaStream_t sq = q == 0 ? c.stream : c.lexs[q - 1];
            if (q > 0) cuda_check(cudaStreamWaitEvent(sq, c.lex_fork, 0), "cudaStreamWaitEvent");
            launch_gs_lex(sq, A, b, inv, dfull, x, forward, mbox_.get() + q * mstride, flags,
                          q > 0 ? prog_.get() + (size_t)(q - 1) * pstride : nullptr,
                          q + 1 < m ? prog_.get() + (size_t)q * pstride : nullptr);
            if (q > 0) cuda_check(cudaEventRecord(c.lex_ev[q - 1], sq), "cudaEventRecord");
        }
        for (int q = 1; q < m; ++q)
            cuda_check(cudaStreamWaitEvent(c.stream, c.lex_ev[q - 1], 0), "cudaStreamWaitEvent");
    }
}

void Hierarchy::vcycle(Ctx& c, int k, const double* b, double* xout, bool zero_in,
                       const MgParams& p, int bt, int* flags, bool* fused_norm)
{
    if (k == kb_) {
        if (cluster_)
            launch_bottom_cluster(c.stream, bottom_args(kb_, bt), b, xout, 1, p.pre, p.post, false,
                                  nullptr, flags);
        else
            launch_bottom(c.stream, bottom_args(kb_, bt), b, xout, 1, p.pre, p.post, false,
                          nullptr, flags);
        return;
    }
    const Op9 A = level_op(k, bt);
    if (lex_) {
        // reference cycle (multigrid.cpp:111-132) with in-place lexicographic sweeps
        if (zero_in) launch_fill(c.stream, xout, 0.0, level_n(k));
        lex_sweeps(c, A, b, k, bt, xout, true, p.pre, flags);
        launch_resid_restrict_tiled(c.stream, A, b, xout, b_[k + 1].get(), xa_[k + 1].get());
        vcycle(c, k + 1, b_[k + 1].get(), xa_[k + 1].get(), true, p, bt, flags);
        launch_prolong_add(c.stream, nx_[k], xa_[k + 1].get(), xout);
        lex_sweeps(c, A, b, k, bt, xout, false, p.post, flags);
        return;
    }
    double* Abuf = xout;
    double* Bbuf = xb_[k].get();
    // sweeps are fused g_sweep_fuse at a time (same colour-pass sequence)
    const int fz = g_sweep_fuse.load(std::memory_order_relaxed);
    const int F = fz < 1 ? 1 : (fz > 5 ? 5 : fz);
    const int Lpre = (p.pre + F - 1) / F, Lpost = (p.post + F - 1) / F;
    const int S = Lpre + Lpost; // out-of-place launches; the last one must land in xout
    auto outbuf = [&](int s) { return ((S - s) % 2 == 0) ? Abuf : Bbuf; };
    const double* cur = zero_in ? nullptr : xout;
    const long long n = level_n(k);
    if (!zero_in && S % 2 == 1) {
        launch_copy(c.stream, xout, Bbuf, n);
        cur = Bbuf;
    }
    int s = 0;
    bool restricted = false; // the last pre-smoothing launch also restricted the residual
    for (int done = 0; done < p.pre;) {
        const int ns = std::min(F, p.pre - done);
        ++s;
        double* out = outbuf(s);
        const bool fuse = g_fuse_restrict.load() && done + ns == p.pre;
        {
            // roofline sample: fine-level launches of the full fusion depth that
            // read x and apply no prolongation (the steady-state launch)
            ProfScope ps(c, (k == 0 && ns == F && cur != nullptr && !fuse) ? kProfSweep : kProfCats);
            restricted = launch_sweep_tiled(c.stream, A, b, inv_at(k, bt), cur, out, true, cur == nullptr,
                                            nullptr, ns, nullptr, nullptr, nullptr, nullptr,
                                            fuse ? b_[k + 1].get() : nullptr, xa_[k + 1].get()) &&
                         fuse;
        }
        cur = out;
        done += ns;
    }
    if (!cur) {
        double* out = outbuf(s);
        launch_fill(c.stream, out, 0.0, n);
        cur = out;
    }
    if (!restricted) launch_resid_restrict_tiled(c.stream, A, b, cur, b_[k + 1].get(), xa_[k + 1].get());
    vcycle(c, k + 1, b_[k + 1].get(), xa_[k + 1].get(), true, p, bt, flags);
    const double* ec = xa_[k + 1].get();
    if (p.post == 0) {
        launch_prolong_add(c.stream, nx_[k], ec, const_cast<double*>(cur));
        return;
    }
    for (int done = 0; done < p.post;) {
        const int ns = std::min(F, p.post - done);
        ++s;
        double* out = outbuf(s);
        // the last launch of the cycle also runs the divergence check if asked
        const bool fuse = fused_norm && done + ns == p.post;
        {
            // the first post launch also applies the prolongation (fused)
            ProfScope ps(c, (k == 0 && done > 0 && ns == F && !fuse) ? kProfSweep : kProfCats);
            const bool f = launch_sweep_tiled(c.stream, A, b, inv_at(k, bt), cur, out, false, false,
                                              done == 0 ? ec : nullptr, ns,
                                              fuse ? part_.get() : nullptr, cnt_.get(),
                                              state_.get(), flags);
            if (fuse) *fused_norm = f;
        }
        cur = out;
        done += ns;
    }
}

void Hierarchy::solve(Ctx& c, const double* b, double* x, const MgParams& p, int bt, int* flags)
{
    const long long n = level_n(0);
    ensure_coarse_op(c, p.pre, p.post); // no-op after Problem::setup_precond (graph capture safe)
    if (kb_ == 0) {
        if (cluster_)
            launch_bottom_cluster(c.stream, bottom_args(0, bt), b, x, p.cycles, p.pre, p.post,
                                  true, state_.get(), flags);
        else
            launch_bottom(c.stream, bottom_args(0, bt), b, x, p.cycles, p.pre, p.post, true,
                          state_.get(), flags);
        launch_check("multigrid bottom solve");
        return;
    }
    if (p.cycles <= 0) {
        launch_fill(c.stream, x, 0.0, n);
        return;
    }
    launch_norm_init(c.stream, b, n, part_.get(), cnt_.get(), state_.get());
    const Op9 A = level_op(0, bt);
    for (int cyc = 0; cyc < p.cycles; ++cyc) {
        bool fused = false; // divergence check run by the cycle's last sweep launch
        vcycle(c, 0, b, x, cyc == 0, p, bt, flags, g_fuse_norm.load() ? &fused : nullptr);
        if (!fused)
            launch_residual_norm_check(c.stream, A, b, x, part_.get(), cnt_.get(), state_.get(), flags);
    }
    launch_check("multigrid solve");
}

bool Hierarchy::can_chain(const MgParams& p, const Op9& M) const
{
    return kb_ == 0 && cluster_ && !lex_ && g_heat_chain.load() && p.cycles > 0 && !M.coef &&
           !M.diag && nx_[0] == 255 && !fine_.coef && fine_.diag && fine_diag_stride_ == level_n(0);
}

bool Hierarchy::solve_chain(Ctx& c, const double* r, double* x, const MgParams& p, int first,
                            int step, int count, const Op9& M, int* flags)
{
    if (!can_chain(p, M) || count <= 0) return false;
    ensure_coarse_op(c, p.pre, p.post);
    ChainArgs ch{};
    ch.nblk = count;
    ch.dbt = step;
    ch.ns = level_n(0);
    for (int d = 0; d < 9; ++d) ch.mc[d] = M.c[d];
    const long long off = (long long)first * ch.ns;
    launch_cluster_chain(c.stream, bottom_args(0, first), r + off, x + off, ch, p.cycles, p.pre,
                         p.post, true, state_.get(), flags);
    launch_check("multigrid chained solve");
    return true;
}

void Hierarchy::smooth(Ctx& c, const double* b, double* x, bool forward, int bt)
{
    const Op9 A = level_op(0, bt);
    DVec inv((size_t)level_n(0)), dfull((size_t)level_n(0));
    launch_inv_diag(c.stream, A, inv.get(), 1, 0, 0, dfull.get());
    if (lex_) {
        DevArray<int> fl(1);
        cudaMemsetAsync(fl.get(), 0, sizeof(int), c.stream);
        launch_gs_lex(c.stream, A, b, inv.get(), dfull.get(), x, forward, mbox_.get(), fl.get());
        c.sync();
        launch_check("smoothing sweep");
        return;
    }
    launch_sweep_tiled(c.stream, A, b, inv.get(), x, xb_[0].get(), forward, false, nullptr, 1);
    launch_copy(c.stream, xb_[0].get(), x, level_n(0));
    c.sync();
    launch_check("smoothing sweep");
}

// ===================================================================== Problem
namespace {

Op9 const_op(int nx, const double c9[9])
{
    Op9 a{};
    a.nx = nx;
    a.coef = nullptr;
    for (int d = 0; d < 9; ++d) a.c[d] = c9[d];
    a.diag = nullptr;
    a.cscale = 1.0;
    return a;
}

Op9 var_op(int nx, const double* coef)
{
    Op9 a{};
    a.nx = nx;
    a.coef = coef;
    a.diag = nullptr;
    a.cscale = 1.0;
    return a;
}

} // namespace

void Problem::upload(DVec& dst, const double* src, size_t n)
{
    dst.resize(n);
    copy_any(ctx, dst.get(), src, n * sizeof(double));
    h2d_bytes_ += (long long)(n * sizeof(double));
}

Problem::Problem(Ctx& c, const oc_problem_desc& d) : ctx(c)
{
    if (d.level < 1 || d.level > 14) throw InvalidArgument("Grid: level out of range");
    if (d.pde < 0 || d.pde > 2) throw InvalidArgument("oc_problem_create: unknown pde");
    // ControlProblem::validate (qp.cpp:10-28)
    if (d.alpha <= 0.0) throw InvalidArgument("ControlProblem: alpha must be positive");
    if (d.beta < 0.0) throw InvalidArgument("ControlProblem: beta must be nonnegative");
    if (!d.u_a || !d.u_b || !d.y_d) throw InvalidArgument("oc_problem_create: missing data");
    if ((d.y_a == nullptr) != (d.y_b == nullptr))
        throw InvalidArgument("ControlProblem: state bounds must come as a pair");
    level_ = d.level;
    nx_ = level_nx(level_);
    ns_ = (long long)nx_ * nx_;
    heat_ = d.pde == OC_PDE_HEAT;
    convdiff_ = d.pde == OC_PDE_CONVDIFF;
    eps_ = d.eps;
    has_sb_ = d.y_a != nullptr;
    partial_obs_ = d.has_obs != 0;

    // (the bound checks of ControlProblem::validate run on the device with the
    // bound splitting below)
    if (partial_obs_) {
        if (d.obs[0] > d.obs[1] || d.obs[2] > d.obs[3])
            throw InvalidArgument("ObservationRegion: empty box");
        if (d.obs[1] < 0.0 || d.obs[0] > 1.0 || d.obs[3] < 0.0 || d.obs[2] > 1.0)
            throw InvalidArgument("ObservationRegion: box outside domain");
    }
    if (convdiff_ && d.eps <= 0.0) throw InvalidArgument("assemble_convdiff: eps must be positive");

    nt_ = 1;
    std::vector<double> qw(1, 1.0);
    if (heat_) {
        if (has_sb_) throw InvalidArgument("assemble_spacetime: state bounds not supported in time");
        if (partial_obs_)
            throw InvalidArgument("assemble_spacetime: partial observation not supported in time");
        if (d.tau <= 0.0) throw InvalidArgument("assemble_spacetime: tau must be positive");
        const double steps = d.horizon / d.tau;
        const long nt = std::lround(steps);
        if (nt < 1 || std::abs(steps - (double)nt) > 1e-9)
            throw InvalidArgument("assemble_spacetime: tau must divide the horizon");
        nt_ = (int)nt;
        qw.assign(nt_, 1.0);
        if (d.quadrature == 1) {
            qw.front() = 0.5;
            qw.back() = 0.5;
        }
    }
    ny_ = ns_ * nt_;
    if (heat_) {
        if (d.y_d_len != ns_ && d.y_d_len != ny_)
            throw InvalidArgument("assemble_spacetime: nodal data size mismatch");
    } else if (d.y_d_len != ns_) {
        throw InvalidArgument("build_qp: nodal data size mismatch with grid");
    }

    // ---- operators (fem.cpp assembly restated in assembly.cpp)
    // grid-constant stencils straight from the element formulas (no level-size
    // assembly on the host; bitwise the centre rows of the full assembly)
    double cM[9];
    stencil9(0, level_, cM);
    P = ProbDev{};
    P.nx = nx_;
    P.ns = ns_;
    P.nt = nt_;
    P.ny = ny_;
    P.heat = heat_ ? 1 : 0;
    P.has_sb = has_sb_ ? 1 : 0;
    P.alpha = d.alpha;
    P.beta = d.beta;
    P.tau = heat_ ? d.tau : 0.0;
    P.M = const_op(nx_, cM);
    P.Mobs = P.M;
    if (convdiff_) {
        // SUPG operator, its transpose and the per-level bases of the
        // rediscretised hierarchies (qp.cpp:143-145), assembled on the device
        Lc_.resize(9 * (size_t)ns_);
        LTc_.resize(9 * (size_t)ns_);
        launch_assemble9(ctx.stream, 2, level_, d.eps, nullptr, Lc_.get());
        launch_transpose9(ctx.stream, nx_, Lc_.get(), LTc_.get());
        P.L = var_op(nx_, Lc_.get());
        P.LT = var_op(nx_, LTc_.get());
        base_.clear();
        baseT_.clear();
        base_.resize(level_ - 1);
        baseT_.resize(level_ - 1);
        for (int k = 0; k + 2 <= level_; ++k) {
            const int l = level_ - k;
            const size_t m9 = 9 * (size_t)level_n(l);
            base_[k].resize(m9);
            baseT_[k].resize(m9);
            if (k == 0) launch_copy(ctx.stream, Lc_.get(), base_[k].get(), (long long)m9);
            else launch_assemble9(ctx.stream, 2, l, d.eps, nullptr, base_[k].get());
            launch_transpose9(ctx.stream, level_nx(l), base_[k].get(), baseT_[k].get());
        }
    } else {
        double cL[9];
        stencil9(1, level_, cL);
        P.L = const_op(nx_, cL);
        P.LT = P.L;
        if (heat_) {
            // Mtl = sparse_add(1, M, 1, tau L) (timedep.cpp:150-153)
            double cMtl[9];
            for (int k = 0; k < 9; ++k) cMtl[k] = 1.0 * cM[k] + 1.0 * (cL[k] * d.tau);
            P.Mtl = const_op(nx_, cMtl);
        }
    }
    if (partial_obs_) {
        Mobsc_.resize(9 * (size_t)ns_);
        launch_assemble9(ctx.stream, 3, level_, 0.0, d.obs, Mobsc_.get());
        P.Mobs = var_op(nx_, Mobsc_.get());
    }

    // ---- problem vectors (build_qp qp.cpp:123-174, assemble_spacetime timedep.cpp:166-213)
    // On the device from the caller's input arrays: only u_a, u_b, y_d (and
    // y_a, y_b, f when given) cross the bus; the split bounds, lumped mass,
    // f = M f_nodal and the time replication are computed here.
    flags_.resize(1);
    cuda_check(cudaMemsetAsync(flags_.get(), 0, sizeof(int), ctx.stream), "memset");
    auto dev_in = [&](const double* src, size_t n, DVec& tmp) -> const double* {
        if (is_device_ptr(src)) return src;
        upload(tmp, src, n);
        return tmp.get();
    };
    DVec t_ua, t_ub, t_f, t_yd;
    const double* dua = dev_in(d.u_a, ns_, t_ua);
    const double* dub = dev_in(d.u_b, ns_, t_ub);
    za_.resize(2 * (size_t)ny_);
    zb_.resize(2 * (size_t)ny_);
    launch_split_bounds(ctx.stream, ns_, nt_, dua, dub, za_.get(), zb_.get(), flags_.get());
    if (has_sb_) {
        upload(ya_, d.y_a, ns_);
        upload(yb_, d.y_b, ns_);
        launch_check_state_bounds(ctx.stream, ns_, ya_.get(), yb_.get(), flags_.get());
    }
    ld_.resize(ns_);
    launch_lumped(ctx.stream, nx_, P.M, ld_.get());
    f_.resize(ny_);
    if (d.f) { // f = M f_nodal (qp.cpp:150), tau-scaled per time block for heat
        DVec mf(ns_);
        launch_op_apply(ctx.stream, P.M, dev_in(d.f, ns_, t_f), mf.get());
        launch_replicate(ctx.stream, ns_, nt_, heat_ ? d.tau : 1.0, mf.get(), f_.get());
        ctx.sync();
    } else {
        launch_fill(ctx.stream, f_.get(), 0.0, ny_);
    }
    if (d.y_d_len == ny_) {
        upload(yd_, d.y_d, ny_);
    } else {
        yd_.resize(ny_);
        launch_replicate(ctx.stream, ns_, nt_, 1.0, dev_in(d.y_d, ns_, t_yd), yd_.get());
    }
    {   // ControlProblem::validate bound checks (qp.cpp:10-28)
        int fl = 0;
        cuda_check(cudaMemcpyAsync(&fl, flags_.get(), sizeof(int), cudaMemcpyDeviceToHost, ctx.stream),
                   "flags");
        ctx.sync();
        if (fl & kErrCtrlBounds)
            throw InvalidArgument("ControlProblem: control bounds must satisfy u_a <= 0 <= u_b");
        if (fl & kErrStateBounds)
            throw InvalidArgument("ControlProblem: state bounds must satisfy y_a <= 0 <= y_b");
    }
    upload(qw_, qw.data(), qw.size());
    P.qw = qw_.get();

    // ---- state, work and scalars
    const size_t N = (size_t)ny_;
    y_.resize(N); z_.resize(2 * N); p_.resize(N);
    lza_.resize(2 * N); lzb_.resize(2 * N); dlza_.resize(2 * N); dlzb_.resize(2 * N);
    if (has_sb_) { lya_.resize(N); lyb_.resize(N); dlya_.resize(N); dlyb_.resize(N); }
    ty_.resize(N); tw_.resize(N); tv_.resize(N);
    rhs_.resize(4 * N); sol_.resize(4 * N);
    mhat_.resize(N); bracket_.resize(N);
    cg_.resize(N); c0_.resize(N); c1_.resize(N); c2_.resize(N);
    t_.resize(N); t2_.resize(N); t3_.resize(N);
    if (heat_) { tf_.resize(N); rblk_.resize((size_t)ns_); }
    part_.resize(8 * kRedBlocks);
    scal_.resize(64);
    flags_.resize(4);
    stop_.resize(2);
    cuda_check(cudaMemsetAsync(flags_.get(), 0, 4 * sizeof(int), ctx.stream), "memset");
    cuda_check(cudaMemsetAsync(stop_.get(), 0, 2 * sizeof(int), ctx.stream), "memset");
    launch_fill(ctx.stream, ty_.get(), 0.0, (long long)N);

    S = IpmDev{};
    S.y = y_.get(); S.z = z_.get(); S.p = p_.get();
    S.lya = lya_.get(); S.lyb = lyb_.get(); S.lza = lza_.get(); S.lzb = lzb_.get();
    S.yd = yd_.get(); S.f = f_.get(); S.za = za_.get(); S.zb = zb_.get();
    S.ya = ya_.get(); S.yb = yb_.get(); S.ld = ld_.get();
    S.ty = ty_.get(); S.tw = tw_.get(); S.tv = tv_.get();
    S.dy = sol_.get(); S.dz = sol_.get() + N; S.dp = sol_.get() + 3 * N;
    S.dlya = dlya_.get(); S.dlyb = dlyb_.get(); S.dlza = dlza_.get(); S.dlzb = dlzb_.get();
    launch_check("problem setup");
    ctx.sync();
}

oc_problem_info Problem::info() const
{
    oc_problem_info i{};
    i.n = (int)ns_;
    i.nt = nt_;
    i.ny = ny_;
    i.kkt_dim = 4 * ny_;
    i.has_state_bounds = has_sb_;
    i.partial_observation = partial_obs_;
    i.symmetric_k = convdiff_ ? 0 : 1;
    i.level = level_;
    i.h2d_bytes = h2d_bytes_;
    return i;
}

void Problem::check_flags(bool sync_now)
{
    if (sync_now) {
        cuda_check(cudaMemcpyAsync(ctx.hflags, flags_.get(), sizeof(int), cudaMemcpyDeviceToHost,
                                   ctx.stream),
                   "flags readback");
        ctx.sync();
    }
    const int f = ctx.hflags[0];
    if (!f) return;
    cudaMemsetAsync(flags_.get(), 0, sizeof(int), ctx.stream);
    if (f & kErrThetaZ) throw RuntimeError("build_theta: lost interiority in z");
    if (f & kErrThetaY) throw RuntimeError("build_theta: lost interiority in y");
    if (f & kErrBadInput) throw InvalidArgument("matching_bracket: inputs must be positive");
    if (f & kErrNegBracket)
        throw RuntimeError(heat_ ? "time_m_hat: negative bracket"
                                 : "matching_bracket: negative bracket entry");
    if (f & kErrSingular2x2) throw RuntimeError("block_2x2_inverse_apply: singular pivot block");
    if (f & kErrMgDiverged)
        throw RuntimeError("MgHierarchy::solve: residual growth, cycle diverged");
    if (f & kErrLexStall) throw RuntimeError("gauss_seidel_sweep: wavefront hand-off stalled");
    if (f & kErrYInterior) throw RuntimeError("ipm: lost strict interiority in y");
    if (f & kErrLamYa) throw RuntimeError("ipm: multiplier not positive in lam_ya");
    if (f & kErrLamYb) throw RuntimeError("ipm: multiplier not positive in lam_yb");
    if (f & kErrZInterior) throw RuntimeError("ipm: lost strict interiority in z");
    if (f & kErrLamZa) throw RuntimeError("ipm: multiplier not positive in lam_za");
    if (f & kErrLamZb) throw RuntimeError("ipm: multiplier not positive in lam_zb");
    throw RuntimeError("device error flag " + std::to_string(f));
}

double Problem::read_scalar(const double* dptr)
{
    cuda_check(cudaMemcpyAsync(ctx.hscal, dptr, sizeof(double), cudaMemcpyDeviceToHost, ctx.stream),
               "scalar readback");
    ctx.sync();
    return ctx.hscal[0];
}

void Problem::set_theta(const double* ty, const double* tw, const double* tv)
{
    if (ty) copy_any(ctx, ty_.get(), ty, ny_ * sizeof(double));
    else launch_fill(ctx.stream, ty_.get(), 0.0, ny_);
    copy_any(ctx, tw_.get(), tw, ny_ * sizeof(double));
    copy_any(ctx, tv_.get(), tv, ny_ * sizeof(double));
}

void Problem::kkt(const double* x, double* out)
{
    launch_kkt(ctx.stream, P, has_sb_ ? ty_.get() : nullptr, tw_.get(), tv_.get(), x, out,
               nullptr, nullptr);
}

void Problem::setup_precond(int kind, const oc_ipm_params& p)
{
    Nvtx nv("precond_setup");
    if (p.cheb_steps < 1) throw InvalidArgument("chebyshev: steps must be >= 1");
    mg_.cycles = p.mg_cycles;
    mg_.pre = p.mg_pre;
    mg_.post = p.mg_post;
    cheb_steps_ = p.cheb_steps;
    if (p.smoother != OC_SMOOTHER_COLOR4 && p.smoother != OC_SMOOTHER_LEX &&
        p.smoother != OC_SMOOTHER_AUTO)
        throw InvalidArgument("ipm: unknown smoother");
    // (a single Newton solve outside ipm_solve has no fallback: AUTO = colour sweeps)
    smoother_ = p.smoother == OC_SMOOTHER_LEX ? OC_SMOOTHER_LEX : OC_SMOOTHER_COLOR4;
    int* fl = flags_.get();
    const double* ty = has_sb_ ? ty_.get() : nullptr;
    if (heat_) {
        // TimeSchurApprox (timedep.cpp:245-261): one hierarchy per time block on
        // M + tau L + diag(mhat_k), built as a batch
        launch_mhat(ctx.stream, P, nullptr, tw_.get(), tv_.get(), mhat_.get(), nullptr, fl);
        Hheat_.allocate(level_, nt_, smoother_);
        Op9 f = P.Mtl;
        f.diag = mhat_.get();
        Hheat_.build(ctx, f, 0, ns_);
    } else if (kind == OC_PRECOND_PPI) {
        // PermutedPrecond (precond.cpp:262-285)
        launch_mhat(ctx.stream, P, nullptr, tw_.get(), tv_.get(), nullptr, bracket_.get(), fl);
        if (!HL_built_ || HL_.smoother() != smoother_) {
            HL_.allocate(level_, 1, smoother_);
            if (convdiff_) {
                std::vector<const double*> b;
                for (auto& v : base_) b.push_back(v.get());
                HL_.build_rediscretized(ctx, P.L, b);
            } else {
                HL_.build(ctx, P.L);
            }
            HL_built_ = true;
        }
        if (!LTpMobs_) {
            // left = L^T + M_obs (+ diag theta_y), sparse_add (precond.cpp:238), assembled
            // on the device from the operators' 9 arrays
            const size_t m9 = 9 * (size_t)ns_;
            DVec lt, mo;
            if (!convdiff_) {
                lt.resize(m9);
                launch_assemble9(ctx.stream, 1, level_, 0.0, nullptr, lt.get());
            }
            if (!partial_obs_) {
                mo.resize(m9);
                launch_assemble9(ctx.stream, 0, level_, 0.0, nullptr, mo.get());
            }
            LTpMobs_.resize(m9);
            launch_add9(ctx.stream, (long long)m9, convdiff_ ? LTc_.get() : lt.get(),
                        partial_obs_ ? Mobsc_.get() : mo.get(), LTpMobs_.get());
            ctx.sync(); // the temporaries return to the pool
        }
        Op9 left = var_op(nx_, LTpMobs_.get());
        left.diag = ty;
        Op9 right = P.L;
        right.diag = bracket_.get();
        Hleft_.allocate(level_, 1, smoother_);
        Hright_.allocate(level_, 1, smoother_);
        if (convdiff_) {
            std::vector<const double*> b, bt;
            for (auto& v : base_) b.push_back(v.get());
            for (auto& v : baseT_) bt.push_back(v.get());
            Hleft_.build_rediscretized(ctx, left, bt);
            Hright_.build_rediscretized(ctx, right, b);
        } else {
            Hleft_.build(ctx, left);
            Hright_.build(ctx, right);
        }
    } else {
        // Block11Approx + SchurApprox (precond.cpp:110-169): F = L + diag(mhat)
        launch_mhat(ctx.stream, P, ty, tw_.get(), tv_.get(), mhat_.get(), nullptr, fl);
        Op9 F = P.L;
        F.diag = mhat_.get();
        HF_.allocate(level_, 1, smoother_);
        if (convdiff_) {
            std::vector<const double*> b, bt;
            for (auto& v : base_) b.push_back(v.get());
            for (auto& v : baseT_) bt.push_back(v.get());
            HF_.build_rediscretized(ctx, F, b);
            Op9 FT = P.LT;
            FT.diag = mhat_.get();
            HFT_.allocate(level_, 1, smoother_);
            HFT_.build_rediscretized(ctx, FT, bt);
        } else {
            HF_.build(ctx, F);
        }
    }
    // dense coarse-cycle operators of the cluster bottom, outside any captured apply
    for (Hierarchy* h : {&Hheat_, &HL_, &Hleft_, &Hright_, &HF_, &HFT_})
        if (h->built()) h->ensure_coarse_op(ctx, mg_.pre, mg_.post);
    setup_kind_ = kind;
    launch_check("preconditioner setup");
}

void Problem::schur_apply(const double* r, double* out)
{
    if (heat_) {
        time_schur(r, out);
        return;
    }
    // SchurApprox::apply_inverse (precond.cpp:130-136)
    int* fl = flags_.get();
    HF_.solve(ctx, r, t2_.get(), mg_, 0, fl);
    launch_schur_middle(ctx.stream, P, has_sb_ ? ty_.get() : nullptr, t2_.get(), t3_.get());
    (convdiff_ ? HFT_ : HF_).solve(ctx, t3_.get(), out, mg_, 0, fl);
}

void Problem::time_schur(const double* r, double* out)
{
    // TimeSchurApprox::apply_inverse (timedep.cpp:268-311)
    int* fl = flags_.get();
    if (Hheat_.can_chain(mg_, P.M)) {
        // each substitution direction as one chained cluster launch (the cluster
        // keeps its SMs for all nt blocks; right-hand sides formed on chip)
        {
            ProfScope ps(ctx, kProfBlock);
            Hheat_.solve_chain(ctx, r, tf_.get(), mg_, 0, 1, nt_, P.M, fl);
        }
        launch_schur_middle(ctx.stream, P, nullptr, tf_.get(), t3_.get());
        ProfScope ps(ctx, kProfBlock);
        Hheat_.solve_chain(ctx, t3_.get(), out, mg_, nt_ - 1, -1, nt_, P.M, fl);
        return;
    }
    for (int k = 0; k < nt_; ++k) {
        const long long off = (long long)k * ns_;
        launch_rhs_plus_mass(ctx.stream, P, r + off, k > 0 ? tf_.get() + off - ns_ : nullptr,
                             rblk_.get());
        ProfScope ps(ctx, kProfBlock);
        Hheat_.solve(ctx, rblk_.get(), tf_.get() + off, mg_, k, fl);
    }
    launch_schur_middle(ctx.stream, P, nullptr, tf_.get(), t3_.get());
    for (int k = nt_ - 1; k >= 0; --k) {
        const long long off = (long long)k * ns_;
        launch_rhs_plus_mass(ctx.stream, P, t3_.get() + off,
                             k + 1 < nt_ ? out + off + ns_ : nullptr, rblk_.get());
        ProfScope ps(ctx, kProfBlock);
        Hheat_.solve(ctx, rblk_.get(), out + off, mg_, k, fl);
    }
}

Problem::~Problem()
{
    cudaStreamSynchronize(ctx.stream);
    drop_graphs();
}

bool graph_reuse();

void Problem::drop_graphs()
{
    for (auto& kv : graphs_) {
        if (!kv.second.exec) continue;
        if (graph_reuse() && ctx.spare_graphs.size() < Ctx::kMaxSpareGraphs)
            ctx.spare_graphs.push_back({kv.second.launches, kv.second.exec});
        else
            cudaGraphExecDestroy(kv.second.exec);
    }
    graphs_.clear();
}

long long Problem::hierarchy_generation() const
{
    return HF_.generation() + HFT_.generation() + HL_.generation() + Hleft_.generation() +
           Hright_.generation() + Hheat_.generation();
}

constexpr long long kMaxGraphLaunches = 2000;

bool graph_reuse()
{
    static const bool on = [] {
        const char* e = getenv("OC_GRAPH_REUSE");
        return !(e && e[0] == '0');
    }();
    return on;
}

// A spare exec of the same length that accepts this graph (same topology and
// kernels; only parameters may differ), or nullptr.
static cudaGraphExec_t take_spare(Ctx& ctx, cudaGraph_t graph, long long launches)
{
    auto& sp = ctx.spare_graphs;
    for (size_t i = sp.size(); i-- > 0;) {
        if (sp[i].launches != launches) continue;
        cudaGraphExecUpdateResultInfo info{};
        if (cudaGraphExecUpdate(sp[i].exec, graph, &info) == cudaSuccess) {
            cudaGraphExec_t e = sp[i].exec;
            sp.erase(sp.begin() + (long)i);
            return e;
        }
        cudaGetLastError(); // topology differs: try the next one
    }
    return nullptr;
}

void Problem::precond_apply(int kind, const double* r, double* out)
{
    static const bool env_off = [] {
        const char* e = getenv("OC_GRAPHS");
        return e && e[0] == '0';
    }();
    // Lexicographic mode runs directly: its applies are tens of milliseconds of
    // wavefront kernels (launch overhead does not matter), GMRES uses every
    // (r, out) pair only once per Newton step, and instantiating the
    // multi-stream graphs of the pipelined sweep batches costs more than their
    // replays save (C3 at 257^2: 26.1 s with graphs, 12.7 s without).
    if (env_off || !graphs_enabled_ || ctx.prof.on || smoother_ == OC_SMOOTHER_LEX) {
        precond_apply_direct(kind, r, out);
        return;
    }
    // the argument checks of precond_apply_direct, which a replay would skip
    if (setup_kind_ < 0) throw InvalidArgument("preconditioner not set up");
    if (kind == OC_PRECOND_PPI) {
        if (heat_) throw InvalidArgument("gmres-ppi is not available for heat problems");
        if (setup_kind_ != OC_PRECOND_PPI) throw InvalidArgument("P_Pi not set up");
    } else if (setup_kind_ == OC_PRECOND_PPI && !heat_) {
        throw InvalidArgument("P_D/P_T not set up");
    }
    // (a tuning change alters launch shapes the captured graphs hold)
    const long long gen = hierarchy_generation() + (g_tuning_gen.load() << 40);
    if (gen != graph_gen_) {
        drop_graphs();
        graph_gen_ = gen;
    }
    // (launch-shape tuning knobs are part of the key: they change the captured launches)
    GraphKey key{kind, r, out, mg_.cycles, mg_.pre, mg_.post, cheb_steps_, g_sweep_tile, g_sweep_fuse};
    GraphEntry& g = graphs_[key];
    if (g.exec) {
        cuda_check(cudaGraphLaunch(g.exec, ctx.stream), "cudaGraphLaunch");
        add_launches(g.launches);
        return;
    }
    if (++g.uses < 2 || g.launches > kMaxGraphLaunches) {
        // first use runs directly (one-time kernel setup, and measures the
        // apply's length); applies of thousands of launches (the heat time
        // substitution) are not worth a graph instantiation
        const long long l0 = t_launches;
        precond_apply_direct(kind, r, out);
        if (g.uses == 1) g.launches = t_launches - l0;
        return;
    }
    const long long l0 = t_launches; // other threads launch concurrently: count our own
    cudaGraph_t graph = nullptr;
    cuda_check(cudaStreamBeginCapture(ctx.stream, cudaStreamCaptureModeThreadLocal),
               "cudaStreamBeginCapture");
    try {
        precond_apply_direct(kind, r, out);
    } catch (...) {
        cudaStreamEndCapture(ctx.stream, &graph);
        if (graph) cudaGraphDestroy(graph);
        throw;
    }
    cuda_check(cudaStreamEndCapture(ctx.stream, &graph), "cudaStreamEndCapture");
    const long long captured = t_launches - l0;
    cudaGraphExec_t exec = graph_reuse() ? take_spare(ctx, graph, captured) : nullptr;
    const cudaError_t e = exec ? cudaSuccess : cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    cuda_check(e, "cudaGraphInstantiate");
    g.exec = exec;
    g.launches = captured;
    add_launches(-captured); // the captured launches did not run; the replay does
    cuda_check(cudaGraphLaunch(exec, ctx.stream), "cudaGraphLaunch");
    add_launches(captured);
}

void Problem::precond_apply_direct(int kind, const double* r, double* out)
{
    if (setup_kind_ < 0) throw InvalidArgument("preconditioner not set up");
    const long long N = ny_;
    const double* ry = r;
    const double* rw = r + N;
    const double* rv = r + 2 * N;
    const double* rp = r + 3 * N;
    double* oy = out;
    double* ow = out + N;
    double* ov = out + 2 * N;
    double* op = out + 3 * N;
    int* fl = flags_.get();
    const double* ty = has_sb_ ? ty_.get() : nullptr;
    if (kind == OC_PRECOND_PPI) {
        if (heat_) throw InvalidArgument("gmres-ppi is not available for heat problems");
        if (setup_kind_ != OC_PRECOND_PPI) throw InvalidArgument("P_Pi not set up");
        // PermutedPrecond::apply (precond.cpp:287-308)
        launch_control_2x2(ctx.stream, P, tw_.get(), tv_.get(), rw, rv, ow, ov, fl);
        launch_ppi_rhs1(ctx.stream, P, ow, ov, rp, t_.get());
        HL_.solve(ctx, t_.get(), oy, mg_, 0, fl);
        launch_ppi_t(ctx.stream, P, ty, oy, ry, t2_.get());
        // SPiHatOperator::apply_inverse (precond.cpp:254-260)
        Hleft_.solve(ctx, t2_.get(), t3_.get(), mg_, 0, fl);
        launch_op_apply(ctx.stream, P.L, t3_.get(), t_.get());
        Hright_.solve(ctx, t_.get(), op, mg_, 0, fl);
        launch_check("P_Pi apply");
        return;
    }
    if (setup_kind_ == OC_PRECOND_PPI && !heat_) throw InvalidArgument("P_D/P_T not set up");
    // BlockDiagPrecond (precond.cpp:202-212) / BlockTriPrecond (:214-230)
    ChebWork w{cg_.get(), c0_.get(), c1_.get(), c2_.get()};
    if (heat_ && kind == OC_PRECOND_PD && g_heat_fork.load()) {
        // P_D's three blocks are independent: the time-block substitution (two
        // chained cluster launches, 256 dependent block solves) runs on the
        // high-priority side stream
        // while Chebyshev and the 2x2 blocks run here; with several solves in
        // flight the priority lets the cluster launches claim their SMs ahead
        // of other solves' wide kernels
        cuda_check(cudaEventRecord(ctx.ev_fork, ctx.stream), "cudaEventRecord");
        cuda_check(cudaStreamWaitEvent(ctx.side, ctx.ev_fork, 0), "cudaStreamWaitEvent");
        std::swap(ctx.stream, ctx.side);
        try {
            schur_apply(rp, op);
        } catch (...) {
            std::swap(ctx.stream, ctx.side);
            throw;
        }
        std::swap(ctx.stream, ctx.side);
        launch_chebyshev(ctx.stream, P, ry, ty, cheb_steps_, w, oy);
        launch_control_2x2(ctx.stream, P, tw_.get(), tv_.get(), rw, rv, ow, ov, fl);
        cuda_check(cudaEventRecord(ctx.ev_join, ctx.side), "cudaEventRecord");
        cuda_check(cudaStreamWaitEvent(ctx.stream, ctx.ev_join, 0), "cudaStreamWaitEvent");
        launch_check("block preconditioner apply");
        return;
    }
    launch_chebyshev(ctx.stream, P, ry, ty, cheb_steps_, w, oy);
    launch_control_2x2(ctx.stream, P, tw_.get(), tv_.get(), rw, rv, ow, ov, fl);
    if (kind == OC_PRECOND_PT) {
        launch_coupling(ctx.stream, P, oy, ow, ov, rp, t_.get());
        schur_apply(t_.get(), op);
    } else {
        schur_apply(rp, op);
    }
    launch_check("block preconditioner apply");
}

void Problem::ensure_krylov(size_t count)
{
    const size_t n4 = 4 * (size_t)ny_;
    bool grew = false;
    while (V_.size() < count + 1) V_.emplace_back(n4);
    while (Z_.size() < count) {
        Z_.emplace_back(n4);
        grew = true;
    }
    if (grew || Ztab_.size() < Z_.size()) {
        std::vector<const double*> tab(Z_.size());
        for (size_t i = 0; i < Z_.size(); ++i) tab[i] = Z_[i].get();
        Ztab_.resize(std::max(Z_.size(), (size_t)1));
        cuda_check(cudaMemcpyAsync(Ztab_.get(), tab.data(), tab.size() * sizeof(const double*),
                                   cudaMemcpyHostToDevice, ctx.stream),
                   "Ztab upload");
        std::vector<const double*> vt(V_.size());
        for (size_t i = 0; i < V_.size(); ++i) vt[i] = V_[i].get();
        Vtab_.resize(V_.size());
        cuda_check(cudaMemcpyAsync(Vtab_.get(), vt.data(), vt.size() * sizeof(const double*),
                                   cudaMemcpyHostToDevice, ctx.stream),
                   "Vtab upload");
        if (!gbar_) {
            gbar_.resize(2);
            cuda_check(cudaMemsetAsync(gbar_.get(), 0, 2 * sizeof(unsigned), ctx.stream), "memset");
        }
        ctx.sync();
    }
}

oc_solve_report Problem::gmres(const oc_ipm_params& p, int kind, const double* b, double* x)
{
    Nvtx nv("gmres");
    // krylov.cpp:133-212 (full GMRES; optional restart every p.gmres_restart)
    oc_solve_report rep{};
    const long long n = 4 * ny_;
    const int maxit = p.linear_maxit;
    const int restart = p.gmres_restart > 0 ? p.gmres_restart : maxit;
    const int ld = std::max(restart, 1) + 1;
    if (H_.size() < (size_t)ld * ld) H_.resize((size_t)ld * ld);
    cs_.resize(ld); sn_.resize(ld); g_.resize(ld); yls_.resize(ld);
    kw_.resize(n); kx2_.resize(n);
    double* scal = scal_.get();
    double* part = part_.get();
    GmresDev G{H_.get(), cs_.get(), sn_.get(), g_.get(), yls_.get(), scal, stop_.get(), ld};

    launch_fill(ctx.stream, x, 0.0, n);
    launch_dot_partials(ctx.stream, b, b, n, part);
    launch_finalize(ctx.stream, part, scal + 0, 1);
    const double bnorm = read_scalar(scal + 0);
    if (bnorm == 0.0) {
        rep.converged = 1;
        return rep;
    }
    double last_relres = 0.0;
    int total = 0;
    bool xbase = false;
    while (total < maxit) {
        // (re)start: r0 = b - A x (restart only), V0 = r0 / ||r0||, g0 = ||r0||
        ensure_krylov(std::min(restart, maxit));
        if (!xbase) {
            launch_scale_inv(ctx.stream, b, scal + 0, V_[0].get(), n, nullptr);
            launch_copy(ctx.stream, scal + 0, g_.get(), 1);
        } else {
            launch_copy(ctx.stream, x, kx2_.get(), n);
            launch_kkt(ctx.stream, P, has_sb_ ? ty_.get() : nullptr, tw_.get(), tv_.get(), x,
                       kw_.get(), nullptr, nullptr);
            // r0 = b - A x (V1 as scratch), V0 = r0 / ||r0||, g0 = ||r0||
            launch_copy(ctx.stream, b, V_[1].get(), n);
            launch_fill(ctx.stream, scal + 6, 1.0, 1);
            launch_axpy_neg(ctx.stream, scal + 6, kw_.get(), V_[1].get(), n);
            launch_dot_partials(ctx.stream, V_[1].get(), V_[1].get(), n, part);
            launch_finalize(ctx.stream, part, scal + 7, 1);
            launch_scale_inv(ctx.stream, V_[1].get(), scal + 7, V_[0].get(), n, nullptr);
            launch_copy(ctx.stream, scal + 7, g_.get(), 1);
        }
        cuda_check(cudaMemsetAsync(stop_.get(), 0, sizeof(int), ctx.stream), "memset");
        for (int j = 0; j < restart && total < maxit; ++j) {
            {
                ProfScope ps(ctx, kProfPrec);
                precond_apply(kind, V_[j].get(), Z_[j].get());
            }
            {
                ProfScope ps(ctx, kProfKkt);
                launch_kkt(ctx.stream, P, has_sb_ ? ty_.get() : nullptr, tw_.get(), tv_.get(),
                           Z_[j].get(), kw_.get(), nullptr, nullptr);
            }
            // modified Gram-Schmidt (krylov.cpp:150-157), each update fused with the
            // next inner product; the last one yields ||w||^2
            double* pa = part; // part_ holds 8 kRedBlocks = 2 kMgsBlocks partials
            double* pb = part + kMgsBlocks;
            const int pmin = g_mgs_persistent.load();
            if (pmin > 0 && j + 1 >= pmin &&
                launch_mgs_persistent(ctx.stream, Vtab_.get(), kw_.get(), G, j, pa, pb, gbar_.get(), n)) {
                if (!(j & 1)) pa = pb; // where step j's partials (||w||^2) landed
            } else {
                launch_dot_partials_mgs(ctx.stream, kw_.get(), V_[0].get(), n, pa);
                for (int i = 0; i <= j; ++i) {
                    const double* next = i < j ? V_[i + 1].get() : kw_.get();
                    launch_mgs_dot(ctx.stream, pa, G, i, j, V_[i].get(), kw_.get(), next, pb, n);
                    std::swap(pa, pb);
                }
            }
            launch_gmres_givens(ctx.stream, pa, G, j);
            launch_scale_inv(ctx.stream, kw_.get(), scal + 1, V_[j + 1].get(), n, stop_.get());
            // The reference rebuilds x and forms the true residual every iteration
            // (krylov.cpp:187-200); neither feeds back into the Krylov iterates, so
            // they are only formed once the residual norm GMRES carries (|g_{j+1}|,
            // equal to ||b - A x_j|| up to rounding) is within 1e3 of the tolerance,
            // and at every exit (cap, restart, exhaustion, zero pivot): same x, same
            // reported residual, same iteration counts.
            bool lazy = g_gmres_lazy_residual.load() != 0;
            if (lazy) {
                launch_gmres_status(ctx.stream, G, j, flags_.get(), scal + 4, scal + 8);
                launch_check("gmres iteration");
                cuda_check(cudaMemcpyAsync(ctx.hscal, scal, 10 * sizeof(double), cudaMemcpyDeviceToHost,
                                           ctx.stream), "readback");
                ctx.sync();
                const double est = ctx.hscal[4] / bnorm;
                const bool last = total + 1 >= maxit || j + 1 >= restart;
                lazy = !(est <= 1e3 * p.linear_tol) && !last && !((int)ctx.hscal[9]) &&
                       !((int)ctx.hscal[8]) && ctx.hscal[1] > 1e-300 && est == est;
                if (lazy) ctx.hscal[2] = est;
            }
            if (!lazy) {
                launch_combine(ctx.stream, Ztab_.get(), yls_.get(), j + 1, x, n,
                               xbase ? kx2_.get() : nullptr);
                launch_kkt(ctx.stream, P, has_sb_ ? ty_.get() : nullptr, tw_.get(), tv_.get(), x,
                           nullptr, b, part);
                // one packed readback: scalars, error flags, stop code
                launch_relres(ctx.stream, part, scal + 0, scal + 2, flags_.get(), stop_.get(), scal + 8);
                launch_check("gmres iteration");
                cuda_check(cudaMemcpyAsync(ctx.hscal, scal, 10 * sizeof(double), cudaMemcpyDeviceToHost,
                                           ctx.stream), "readback");
                ctx.sync();
            }
            ctx.hflags[0] = (int)ctx.hscal[8];
            ctx.hflags[1] = (int)ctx.hscal[9];
            check_flags(false);
            const double hnext = ctx.hscal[1];
            const double relres = ctx.hscal[2];
            if (ctx.hflags[1]) {
                // zero pivot: the reference breaks before rebuilding x (krylov.cpp:166-170)
                std::snprintf(rep.message, sizeof(rep.message),
                              "gmres: zero pivot in Hessenberg triangularization");
                if (j > 0)
                    launch_combine(ctx.stream, Ztab_.get(), yls_.get(), j, x, n,
                                   xbase ? kx2_.get() : nullptr);
                else if (xbase)
                    launch_copy(ctx.stream, kx2_.get(), x, n);
                else
                    launch_fill(ctx.stream, x, 0.0, n);
                rep.relative_residual = last_relres;
                return rep;
            }
            ++total;
            rep.iterations = total;
            rep.relative_residual = relres;
            last_relres = relres;
            if (relres <= p.linear_tol) {
                rep.converged = 1;
                return rep;
            }
            if (hnext <= 1e-300) {
                std::snprintf(rep.message, sizeof(rep.message),
                              "gmres: Krylov space exhausted before tolerance");
                return rep;
            }
        }
        xbase = true; // restart from the current iterate
    }
    std::snprintf(rep.message, sizeof(rep.message), "gmres: max iterations reached");
    return rep;
}

oc_solve_report Problem::minres(const oc_ipm_params& p, int kind, const double* b, double* x)
{
    Nvtx nv("minres");
    // krylov.cpp:37-131
    oc_solve_report rep{};
    const long long n = 4 * ny_;
    for (auto& v : kvec_) v.resize(n);
    kw_.resize(n);
    double* vprev = kvec_[0].get();
    double* v = kvec_[1].get();
    double* vnext = kvec_[2].get();
    double* z = kvec_[3].get();
    double* znext = kvec_[4].get();
    double* wprev = kvec_[5].get();
    double* w = kvec_[6].get();
    double* wnext = kvec_[7].get();
    double* az = kw_.get();
    double* sc = scal_.get() + 16; // MINRES scalar slots
    double* part = part_.get();
    int* stop = stop_.get();

    launch_fill(ctx.stream, x, 0.0, n);
    launch_dot_partials(ctx.stream, b, b, n, part);
    launch_finalize(ctx.stream, part, scal_.get() + 0, 1);
    const double bnorm = read_scalar(scal_.get() + 0);
    if (bnorm == 0.0) {
        rep.converged = 1;
        return rep;
    }
    launch_fill(ctx.stream, vprev, 0.0, n);
    launch_copy(ctx.stream, b, v, n);
    precond_apply(kind, v, z);
    launch_dot_partials(ctx.stream, z, v, n, part);
    launch_minres_setup(ctx.stream, part, sc);
    cuda_check(cudaMemsetAsync(stop, 0, sizeof(int), ctx.stream), "memset");
    const double gamma_sq = read_scalar(sc + 15);
    check_flags(true);
    if (!(gamma_sq > 0.0)) {
        rep.breakdown = 1;
        std::snprintf(rep.message, sizeof(rep.message),
                      "minres: preconditioner not positive definite");
        rep.relative_residual = 1.0;
        return rep;
    }
    launch_fill(ctx.stream, wprev, 0.0, n);
    launch_fill(ctx.stream, w, 0.0, n);
    const double* tyk = has_sb_ ? ty_.get() : nullptr;
    for (int j = 1; j <= p.linear_maxit; ++j) {
        launch_scale_inv(ctx.stream, z, sc + 0, z, n, nullptr);
        {
            ProfScope ps(ctx, kProfKkt);
            launch_kkt(ctx.stream, P, tyk, tw_.get(), tv_.get(), z, az, nullptr, nullptr);
        }
        launch_dot_partials(ctx.stream, az, z, n, part);
        launch_minres_delta(ctx.stream, part, sc);
        launch_minres_vnext(ctx.stream, az, v, vprev, vnext, sc, j == 1 ? 1 : 0, n);
        {
            ProfScope ps(ctx, kProfPrec);
            precond_apply(kind, vnext, znext);
        }
        launch_dot_partials(ctx.stream, znext, vnext, n, part);
        launch_minres_gamma(ctx.stream, part, sc, stop);
        launch_minres_update(ctx.stream, z, wprev, w, wnext, x, sc, stop, n);
        launch_minres_rotate(ctx.stream, sc, stop);
        launch_kkt(ctx.stream, P, tyk, tw_.get(), tv_.get(), x, nullptr, b, part);
        // one packed readback per iteration: scalars, error flags, stop code
        launch_relres(ctx.stream, part, scal_.get() + 0, scal_.get() + 2, flags_.get(), stop,
                      scal_.get() + 8);
        launch_check("minres iteration");
        cuda_check(cudaMemcpyAsync(ctx.hscal, scal_.get(), 17 * sizeof(double), // + gamma (sc[0])
                                   cudaMemcpyDeviceToHost, ctx.stream), "readback");
        ctx.sync();
        ctx.hflags[0] = (int)ctx.hscal[8];
        ctx.hflags[1] = (int)ctx.hscal[9];
        check_flags(false);
        const double relres = ctx.hscal[2];
        const int st = ctx.hflags[1];
        if (st == 1) {
            rep.breakdown = 1;
            std::snprintf(rep.message, sizeof(rep.message),
                          "minres: preconditioner lost definiteness");
            rep.iterations = j;
            rep.relative_residual = relres;
            return rep;
        }
        if (st == 2) {
            rep.iterations = j;
            rep.relative_residual = relres;
            rep.converged = relres <= p.linear_tol;
            return rep;
        }
        std::swap(vprev, v);
        std::swap(v, vnext);
        std::swap(z, znext);
        std::swap(wprev, w);
        std::swap(w, wnext);
        rep.iterations = j;
        rep.relative_residual = relres;
        if (relres <= p.linear_tol) {
            rep.converged = 1;
            return rep;
        }
        if (ctx.hscal[16 + 0] == 0.0) break; // gamma == 0: Krylov space exhausted
    }
    if (!rep.converged) std::snprintf(rep.message, sizeof(rep.message), "minres: max iterations reached");
    return rep;
}

oc_solve_report Problem::newton_solve(const oc_ipm_params& p, const double* rhs, double* x)
{
    int kind;
    bool use_gmres;
    if (heat_) {
        // make_spacetime_model supports gmres-pt (timedep.cpp:344-431); the
        // block-diagonal MINRES variant is the BASELINE config-5 extension.
        if (p.solver == OC_SOLVER_GMRES_PT) { kind = OC_PRECOND_PT; use_gmres = true; }
        else if (p.solver == OC_SOLVER_MINRES_PD) { kind = OC_PRECOND_PD; use_gmres = false; }
        else throw InvalidArgument("spacetime newton_solve: unsupported solver kind");
    } else {
        switch (p.solver) {
        case OC_SOLVER_MINRES_PD:
            if (partial_obs_) throw InvalidArgument("minres-pd requires a nonsingular (1,1) block");
            kind = OC_PRECOND_PD; use_gmres = false; break;
        case OC_SOLVER_GMRES_PT:
            if (partial_obs_) throw InvalidArgument("gmres-pt requires a nonsingular (1,1) block");
            kind = OC_PRECOND_PT; use_gmres = true; break;
        case OC_SOLVER_GMRES_PPI:
            kind = OC_PRECOND_PPI; use_gmres = true; break;
        default:
            throw InvalidArgument("newton_solve: the dense solver is a CPU verification path");
        }
    }
    setup_precond(kind, p);
    return use_gmres ? gmres(p, kind, rhs, x) : minres(p, kind, rhs, x);
}

void Problem::ipm_solve(const oc_ipm_params& p, oc_ipm_result* r)
{
    Nvtx nv("ipm_solve");
    // ipm_solve (ipm.cpp:270-341)
    if (!(p.alpha0 > 0.0 && p.alpha0 < 1.0))
        throw InvalidArgument("ipm_solve: alpha0 must lie in (0,1)");
    if (!(p.sigma > 0.0 && p.sigma < 1.0)) throw InvalidArgument("ipm_solve: sigma must lie in (0,1)");
    if (p.mu0 <= 0.0) throw InvalidArgument("ipm_solve: mu0 must be positive");
    cudaEvent_t es, ee, ns, ne;
    cuda_check(cudaEventCreate(&es), "event");
    cuda_check(cudaEventCreate(&ee), "event");
    cuda_check(cudaEventCreate(&ns), "event");
    cuda_check(cudaEventCreate(&ne), "event");
    struct EvGuard {
        cudaEvent_t* e;
        ~EvGuard() { for (int i = 0; i < 4; ++i) cudaEventDestroy(e[i]); }
    };
    cudaEvent_t evs[4] = {es, ee, ns, ne};
    EvGuard guard{evs};

    cuda_check(cudaMemsetAsync(flags_.get(), 0, sizeof(int), ctx.stream), "memset");
    cudaEventRecord(es, ctx.stream);
    launch_initial_point(ctx.stream, P, S);
    double* norms = scal_.get() + 40;
    double* steps = scal_.get() + 44;
    launch_ipm_residuals(ctx.stream, P, S, p.mu0, part_.get(), norms);
    cuda_check(cudaMemcpyAsync(ctx.hscal, norms, 3 * sizeof(double), cudaMemcpyDeviceToHost,
                               ctx.stream), "readback");
    ctx.sync();
    double nrm[3] = {ctx.hscal[0], ctx.hscal[1], ctx.hscal[2]};
    std::vector<oc_iter_record> recs;
    recs.push_back({0, p.mu0, nrm[0], nrm[1], nrm[2], 0, 0.0, 1, 0.0});

    double state_mu = p.mu0;
    int k = 0;
    auto converged = [&]() {
        return nrm[0] <= p.eps_p && nrm[1] <= p.eps_d && nrm[2] <= p.eps_c && state_mu <= p.eps_c;
    };
    double mu = p.mu0;
    long long total_lin = 0, discarded_lin = 0;
    double newton_total = 0.0;
    // AUTO smoother: colour sweeps until a Newton solve is capped, then the
    // lexicographic smoother from that step on (the capped solve is redone)
    oc_ipm_params pp = p;
    const bool autosm = p.smoother == OC_SMOOTHER_AUTO;
    if (autosm) pp.smoother = OC_SMOOTHER_COLOR4;
    int lex_from = p.smoother == OC_SMOOTHER_LEX ? 1 : 0;
    while (!converged() && k < p.max_iterations) {
        mu = p.sigma * mu;
        launch_theta(ctx.stream, P, S, flags_.get());
        launch_newton_rhs(ctx.stream, P, S, mu, rhs_.get());
        cudaEventRecord(ns, ctx.stream);
        oc_solve_report rep = newton_solve(pp, rhs_.get(), sol_.get());
        if (autosm && pp.smoother == OC_SMOOTHER_COLOR4 && !rep.converged &&
            rep.iterations >= p.linear_maxit) {
            discarded_lin += rep.iterations;
            pp.smoother = OC_SMOOTHER_LEX;
            lex_from = k + 1;
            rep = newton_solve(pp, rhs_.get(), sol_.get());
        }
        cudaEventRecord(ne, ctx.stream);
        launch_recover_ratios(ctx.stream, P, S, mu, part_.get());
        launch_step_lengths(ctx.stream, part_.get(), p.alpha0, steps);
        launch_ipm_update(ctx.stream, P, S, steps, flags_.get());
        state_mu = mu;
        ++k;
        launch_ipm_residuals(ctx.stream, P, S, mu, part_.get(), norms);
        launch_check("ipm iteration");
        cuda_check(cudaMemcpyAsync(ctx.hscal, norms, 3 * sizeof(double), cudaMemcpyDeviceToHost,
                                   ctx.stream), "readback");
        cuda_check(cudaMemcpyAsync(ctx.hflags, flags_.get(), sizeof(int), cudaMemcpyDeviceToHost,
                                   ctx.stream), "readback");
        ctx.sync();
        check_flags(false);
        float nms = 0.f;
        cudaEventElapsedTime(&nms, ns, ne);
        newton_total += nms;
        nrm[0] = ctx.hscal[0];
        nrm[1] = ctx.hscal[1];
        nrm[2] = ctx.hscal[2];
        total_lin += rep.iterations;
        recs.push_back({k, mu, nrm[0], nrm[1], nrm[2], rep.iterations, rep.relative_residual,
                        rep.converged, (double)nms});
    }
    const bool conv = converged();
    // outputs: objective, sparsity, vectors
    double* obj = scal_.get() + 48;
    launch_objective(ctx.stream, P, S, part_.get(), obj);
    cudaEventRecord(ee, ctx.stream);
    cuda_check(cudaMemcpyAsync(ctx.hscal, obj, 3 * sizeof(double), cudaMemcpyDeviceToHost,
                               ctx.stream), "readback");
    ctx.sync();
    float sms = 0.f;
    cudaEventElapsedTime(&sms, es, ee);
    r->objective = ctx.hscal[0];
    const double below = ctx.hscal[1];
    r->l1 = ctx.hscal[2];
    r->sparsity_pct = ny_ == 0 ? 100.0 : 100.0 * below / (double)ny_;
    const long long all = (long long)(nx_ + 2) * (nx_ + 2);
    r->nodal_sparsity_pct =
        100.0 * (below + (double)((all - ns_) * nt_)) / (double)(all * nt_);
    r->nli = k;
    r->converged = conv ? 1 : 0;
    r->av_li = k > 0 ? (double)total_lin / k : 0.0;
    r->total_lin = total_lin;
    r->mu = state_mu;
    r->solve_ms = sms;
    r->newton_ms = newton_total;
    r->discarded_lin = discarded_lin;
    r->lex_from = lex_from;
    r->n_records = (int)recs.size();
    if (r->records)
        for (int i = 0; i < std::min(r->n_records, r->records_cap); ++i) r->records[i] = recs[i];
    const size_t N = (size_t)ny_;
    if (r->y) copy_any(ctx, r->y, y_.get(), N * sizeof(double));
    if (r->z) copy_any(ctx, r->z, z_.get(), 2 * N * sizeof(double));
    if (r->p) copy_any(ctx, r->p, p_.get(), N * sizeof(double));
    if (r->lam_za) copy_any(ctx, r->lam_za, lza_.get(), 2 * N * sizeof(double));
    if (r->lam_zb) copy_any(ctx, r->lam_zb, lzb_.get(), 2 * N * sizeof(double));
    if (has_sb_) {
        if (r->lam_ya) copy_any(ctx, r->lam_ya, lya_.get(), N * sizeof(double));
        if (r->lam_yb) copy_any(ctx, r->lam_yb, lyb_.get(), N * sizeof(double));
    }
    if (r->u) {
        launch_recover_control(ctx.stream, ny_, z_.get(), t_.get());
        copy_any(ctx, r->u, t_.get(), N * sizeof(double));
    }
    ctx.sync();
}

void Problem::ipm_pieces(const double* y, const double* z, const double* pv, const double* lya,
                         const double* lyb, const double* lza, const double* lzb, double mu_state,
                         double mu_rhs, double* ty, double* tw, double* tv, double* r1, double* r2,
                         double* r3, double* norms3)
{
    const size_t N = (size_t)ny_;
    copy_any(ctx, y_.get(), y, N * 8);
    copy_any(ctx, z_.get(), z, 2 * N * 8);
    copy_any(ctx, p_.get(), pv, N * 8);
    copy_any(ctx, lza_.get(), lza, 2 * N * 8);
    copy_any(ctx, lzb_.get(), lzb, 2 * N * 8);
    if (has_sb_) {
        copy_any(ctx, lya_.get(), lya, N * 8);
        copy_any(ctx, lyb_.get(), lyb, N * 8);
    }
    cuda_check(cudaMemsetAsync(flags_.get(), 0, sizeof(int), ctx.stream), "memset");
    launch_theta(ctx.stream, P, S, flags_.get());
    launch_newton_rhs(ctx.stream, P, S, mu_rhs, rhs_.get());
    double* norms = scal_.get() + 40;
    launch_ipm_residuals(ctx.stream, P, S, mu_state, part_.get(), norms);
    if (ty) {
        if (has_sb_) copy_any(ctx, ty, ty_.get(), N * 8);
        else {
            launch_fill(ctx.stream, t_.get(), 0.0, ny_);
            copy_any(ctx, ty, t_.get(), N * 8);
        }
    }
    if (tw) copy_any(ctx, tw, tw_.get(), N * 8);
    if (tv) copy_any(ctx, tv, tv_.get(), N * 8);
    if (r1) copy_any(ctx, r1, rhs_.get(), N * 8);
    if (r2) copy_any(ctx, r2, rhs_.get() + N, 2 * N * 8);
    if (r3) copy_any(ctx, r3, rhs_.get() + 3 * N, N * 8);
    cuda_check(cudaMemcpyAsync(ctx.hscal, norms, 3 * sizeof(double), cudaMemcpyDeviceToHost,
                               ctx.stream), "readback");
    ctx.sync();
    if (norms3) std::memcpy(norms3, ctx.hscal, 3 * sizeof(double));
    check_flags(true);
}

double Problem::objective(const double* y, const double* z)
{
    const size_t N = (size_t)ny_;
    copy_any(ctx, y_.get(), y, N * 8);
    copy_any(ctx, z_.get(), z, 2 * N * 8);
    double* obj = scal_.get() + 48;
    launch_objective(ctx.stream, P, S, part_.get(), obj);
    return read_scalar(obj);
}

void Problem::time_applies(int kind, int reps, double* kkt_ms, double* prec_ms)
{
    if (setup_kind_ < 0) throw InvalidArgument("preconditioner not set up");
    const long long n = 4 * ny_;
    kw_.resize(n);
    kx2_.resize(n);
    launch_fill(ctx.stream, kx2_.get(), 1.0, n);
    // warm-up (two preconditioner applies: the second one captures its graph)
    kkt(kx2_.get(), kw_.get());
    precond_apply(kind, kx2_.get(), kw_.get());
    precond_apply(kind, kx2_.get(), kw_.get());
    ctx.sync();
    cudaEventRecord(ctx.ev0, ctx.stream);
    for (int i = 0; i < reps; ++i) kkt(kx2_.get(), kw_.get());
    cudaEventRecord(ctx.ev1, ctx.stream);
    ctx.sync();
    float a = 0.f;
    cudaEventElapsedTime(&a, ctx.ev0, ctx.ev1);
    cudaEventRecord(ctx.ev0, ctx.stream);
    const auto h0 = std::chrono::steady_clock::now();
    for (int i = 0; i < reps; ++i) precond_apply(kind, kx2_.get(), kw_.get());
    cudaEventRecord(ctx.ev1, ctx.stream);
    const auto h1 = std::chrono::steady_clock::now();
    ctx.sync();
    if (std::getenv("OC_DEBUG_HOST_TIME")) // tuning aid: host enqueue time vs device time
        std::fprintf(stderr, "precond apply host enqueue %.3f ms\n",
                     std::chrono::duration<double, std::milli>(h1 - h0).count() / reps);
    float b = 0.f;
    cudaEventElapsedTime(&b, ctx.ev0, ctx.ev1);
    *kkt_ms = a / reps;
    *prec_ms = b / reps;
    check_flags(true);
}

} // namespace ocb
