// Krylov vector kernels (sm_100a, FP64): deterministic reductions, the MGS
// Arnoldi step, GMRES Givens/back-substitution and the MINRES recurrences.
//
// Reductions use a fixed grid of kRedBlocks partials summed in a fixed order,
// so repeated solves are bit-identical (reference kernels.hpp:20-21). The
// scalar recurrences run in one thread on the device so the host only reads
// the convergence scalars once per Krylov iteration.
#include "kernels.hpp"

#include <stdexcept>
#include <string>

namespace ocb {

namespace {

constexpr int kT = 256;
inline unsigned blocks_for(long long n) { return (unsigned)((n + kT - 1) / kT); }

__global__ void __launch_bounds__(kRedThreads) k_dot_partials(const double* __restrict__ x,
                                                              const double* __restrict__ y,
                                                              long long n, double* __restrict__ part)
{
    __shared__ double sh[32];
    double acc = 0.0;
    // unrolled so several loads are in flight; the accumulation order is unchanged
#pragma unroll 4
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        acc += x[i] * y[i];
    acc = block_sum(acc, sh);
    if (threadIdx.x == 0) part[blockIdx.x] = acc;
}

__global__ void k_finalize(const double* __restrict__ part, double* dst, int mode)
{
    const double s = sum_partials_warp(part, kRedBlocks);
    if (threadIdx.x == 0) dst[0] = mode == 1 ? sqrt(s) : s;
}

__global__ void k_copy(const double* __restrict__ x, double* __restrict__ y, long long n)
{
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) y[i] = x[i];
}

__global__ void k_fill(double* __restrict__ x, double v, long long n)
{
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) x[i] = v;
}

__global__ void k_scale_inv(const double* x, const double* __restrict__ den, double* y,
                            long long n, const int* __restrict__ stop)
{
    if (stop && *stop) return;
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const double d = *den;
    if (stop && !(d > 1e-300)) return; // GMRES: basis exhausted, V_{j+1} not formed
    if (i < n) y[i] = x[i] * (1.0 / d);
}

__global__ void k_axpy_neg(const double* __restrict__ h, const double* __restrict__ v,
                           double* __restrict__ w, long long n)
{
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) w[i] += (-h[0]) * v[i];
}

__global__ void k_combine(const double* const* __restrict__ Z, const double* __restrict__ y,
                          int m, double* __restrict__ x, long long n, const double* __restrict__ xb)
{
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double acc = xb ? xb[i] : 0.0;
#pragma unroll 4
    for (int k = 0; k < m; ++k) acc += y[k] * Z[k][i]; // loads in flight, order unchanged
    x[i] = acc;
}

__global__ void k_add(const double* __restrict__ a, const double* __restrict__ b,
                      double* __restrict__ out, long long n)
{
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = a[i] + b[i];
}

__global__ void k_mgs_step(const double* __restrict__ part, double* H, int ld, int i, int j,
                           const double* __restrict__ vi, double* __restrict__ w, long long n)
{
    __shared__ double hs;
    if (threadIdx.x < 32) {
        const double s = sum_partials_warp(part, kRedBlocks);
        if (threadIdx.x == 0) {
            hs = s;
            if (blockIdx.x == 0) H[(long long)j * ld + i] = s;
        }
    }
    __syncthreads();
    const double h = hs;
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < n;
         k += (long long)gridDim.x * blockDim.x)
        w[k] += (-h) * vi[k];
}

// Modified Gram-Schmidt step i fused with the next dot product: h_ij = sum of
// the kMgsBlocks partials part_in (fixed order), w -= h_ij v_i, and the
// kMgsBlocks partials of <w, vnext> into part_out (one pass over w less than a
// separate update + dot; a wider grid than kRedBlocks for memory parallelism).
__global__ void __launch_bounds__(kRedThreads) k_mgs_dot(const double* __restrict__ part_in,
                                                         double* H, int ld, int i, int j,
                                                         const double* __restrict__ vi,
                                                         double* __restrict__ w,
                                                         const double* vnext,
                                                         double* __restrict__ part_out, long long n)
{
    __shared__ double hs;
    __shared__ double sh[32];
    if (threadIdx.x < 32) {
        const double s = sum_partials_warp(part_in, kMgsBlocks);
        if (threadIdx.x == 0) {
            hs = s;
            if (blockIdx.x == 0) H[(long long)j * ld + i] = s;
        }
    }
    __syncthreads();
    const double h = hs;
    double acc = 0.0;
#pragma unroll 4
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < n;
         k += (long long)gridDim.x * blockDim.x) {
        const double wn = w[k] + (-h) * vi[k];
        w[k] = wn;
        acc += wn * (vnext == w ? wn : vnext[k]);
    }
    acc = block_sum(acc, sh);
    if (threadIdx.x == 0) part_out[blockIdx.x] = acc;
}

// Whole modified Gram-Schmidt orthogonalisation of GMRES column j in ONE
// persistent launch (one 1024-thread CTA per SM, co-resident by cooperative
// launch): w stays in shared memory for all j+1 steps, so each step streams
// only v_i and v_{i+1} instead of reading and writing w as well
// (k_dot_partials_mgs + j+1 k_mgs_dot launches move 4 vectors per step).
// Bitwise identical to that sequence: the kMgsBlocks "virtual blocks" keep
// their element sets (k = b*256 + t + m*kMgsBlocks*256), each thread
// accumulates over m in the same order, the 256-thread block sum and the
// fixed-order partial sums are the same functions; a grid barrier replaces
// the kernel boundary between steps. Partials alternate between pa and pb;
// the last step's (||w||^2) land in pfinal.
constexpr int kMgsPersistThreads = 1024;
constexpr int kMgsPersistM = 14; // elements per virtual-block thread held on chip
static_assert(kMgsPersistM % 7 == 0, "loads are batched 7 at a time");
constexpr int kMgsSmemM = kMgsPersistM - 1; // slices of w in shared memory (the last in global)

__device__ __forceinline__ double ld_l2_hint(const double* p, unsigned long long pol)
{
    double v;
    asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;\n" : "=d"(v) : "l"(p), "l"(pol));
    return v;
}

// L2 prefetch of this CTA's chunks of a basis vector (one 2 KB block per
// virtual block and m slice; the ragged end rounds down to 16 bytes)
__device__ __forceinline__ void prefetch_chunks(const double* v, int vb0, int vpb, long long n)
{
    const long long stride = (long long)kMgsBlocks * 256;
    for (int q = threadIdx.x; q < vpb * kMgsPersistM; q += blockDim.x) {
        const long long k = (long long)(vb0 + q / kMgsPersistM) * 256 + (q % kMgsPersistM) * stride;
        if (k >= n) continue;
        const unsigned bytes = (unsigned)(min(256LL, n - k) * 8) & ~15u;
        if (bytes)
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(v + k), "r"(bytes) : "memory");
    }
}

__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p)
{
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Grid barrier over co-resident CTAs: bar[0] arrivals, bar[1] generation.
// Release on arrival (the CTA's writes, ordered by the bar.sync before it),
// acquire on the generation poll.
__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned nblocks)
{
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned g = ld_acquire_gpu(bar + 1);
        unsigned old;
        asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;\n" : "=r"(old) : "l"(bar) : "memory");
        if (old == nblocks - 1) {
            asm volatile("st.relaxed.gpu.global.u32 [%0], 0;\n" ::"l"(bar) : "memory");
            asm volatile("red.release.gpu.global.add.u32 [%0], 1;\n" ::"l"(bar + 1) : "memory");
        } else {
            while (ld_acquire_gpu(bar + 1) == g) {
            }
        }
    }
    __syncthreads();
}

__global__ void __launch_bounds__(kMgsPersistThreads, 1)
    k_mgs_persistent(const double* const* __restrict__ V, double* __restrict__ w, double* H, int ld,
                     int j, double* pa, double* pb, double* pfinal, unsigned* bar, long long n)
{
    // dynamic: ps[kMgsBlocks] partials, then ws[local vb][m < kMgsSmemM][t]; the
    // last m slice of w (the ragged tail) stays in global memory
    extern __shared__ double dyn[];
    double* ps = dyn;
    double* ws = dyn + kMgsBlocks;
    __shared__ double sh[32];
    __shared__ double hs;
    constexpr int GT = 256, GROUPS = kMgsPersistThreads / GT;
    const int vpb = kMgsBlocks / gridDim.x; // virtual blocks per CTA
    const int g = threadIdx.x / GT, t = threadIdx.x % GT;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, gw = wid % (GT / 32);
    const long long stride = (long long)kMgsBlocks * GT;

    // block_sum restricted to one virtual block's 8 warps (block_sum's order)
    auto vb_sum = [&](double acc) {
        acc = warp_sum(acc);
        __syncthreads();
        if (lane == 0) sh[wid] = acc;
        __syncthreads();
        double v = (lane < GT / 32 && gw == 0) ? sh[(wid / (GT / 32)) * (GT / 32) + lane] : 0.0;
        if (gw == 0) v = warp_sum(v);
        return v;
    };

    // stage w, then the first inner product <w, v_0> (k_dot_partials on kMgsBlocks)
    if (j >= 1) prefetch_chunks(V[1], blockIdx.x * vpb, vpb, n);
    for (int s = g; s < vpb; s += GROUPS) {
        const int vb = blockIdx.x * vpb + s;
        double* wl = ws + (size_t)s * kMgsSmemM * GT + t;
        double acc = 0.0;
        const double* v0 = V[0];
#pragma unroll 2
        for (int m = 0; m < kMgsPersistM; ++m) {
            const long long k = (long long)vb * GT + t + m * stride;
            if (k < n) {
                const double x = w[k];
                if (m < kMgsSmemM) wl[m * GT] = x;
                acc += x * v0[k];
            }
        }
        const double v = vb_sum(acc);
        if (t == 0) pa[vb] = v;
    }
    for (int i = 0; i <= j; ++i) {
        double* pin = (i & 1) ? pb : pa;
        double* pout = i == j ? pfinal : ((i & 1) ? pa : pb);
        // the step after this one streams v_{i+2}: start it towards L2 now (the
        // basis vectors do not depend on the reductions)
        if (i + 2 <= j) prefetch_chunks(V[i + 2], blockIdx.x * vpb, vpb, n);
        grid_barrier(bar, gridDim.x);
        // the partials through L2 into shared memory (one round trip), then
        // sum_partials_warp's order from there
        for (int q = threadIdx.x; q < kMgsBlocks; q += kMgsPersistThreads) ps[q] = __ldcg(pin + q);
        __syncthreads();
        if (threadIdx.x < 32) {
            double s = 0.0;
#pragma unroll 8
            for (int q = lane; q < kMgsBlocks; q += 32) s += ps[q];
            s = warp_sum(s);
            if (threadIdx.x == 0) {
                hs = s;
                if (blockIdx.x == 0) H[(long long)j * ld + i] = s;
            }
        }
        __syncthreads();
        const double h = hs;
        // v_{i+1} is read again as v_i by the next step: keep it in L2, let v_i go
        unsigned long long pol_first, pol_last;
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol_first));
        asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(pol_last));
        const double* __restrict__ vi = V[i];
        const double* __restrict__ vn = i < j ? V[i + 1] : nullptr;
        for (int s = g; s < vpb; s += GROUPS) {
            const int vb = blockIdx.x * vpb + s;
            double* wl = ws + (size_t)s * kMgsSmemM * GT + t;
            double acc = 0.0;
            // valid elements form a prefix m < mc; loads of 7 elements are issued
            // before their updates (the order of acc is unchanged)
            const long long k0 = (long long)vb * GT + t;
            const int mc = k0 < n ? (int)min((long long)kMgsPersistM, (n - 1 - k0) / stride + 1) : 0;
#pragma unroll
            for (int m0 = 0; m0 < kMgsPersistM; m0 += 7) {
                double a[7], c[7];
#pragma unroll
                for (int u = 0; u < 7; ++u) {
                    const long long k = k0 + (m0 + u) * stride;
                    a[u] = m0 + u < mc ? ld_l2_hint(vi + k, pol_first) : 0.0;
                    c[u] = (vn && m0 + u < mc) ? ld_l2_hint(vn + k, pol_last) : 0.0;
                }
#pragma unroll
                for (int u = 0; u < 7; ++u) {
                    const int m = m0 + u;
                    if (m < mc) {
                        double* wp = m < kMgsSmemM ? wl + m * GT : w + (k0 + m * stride);
                        const double wn = *wp + (-h) * a[u];
                        *wp = wn;
                        acc += wn * (vn ? c[u] : wn);
                    }
                }
            }
            const double v = vb_sum(acc);
            if (t == 0) pout[vb] = v;
        }
    }
    for (int s = g; s < vpb; s += GROUPS) {
        const int vb = blockIdx.x * vpb + s;
        const double* wl = ws + (size_t)s * kMgsSmemM * GT + t;
        for (int m = 0; m < kMgsSmemM; ++m) {
            const long long k = (long long)vb * GT + t + m * stride;
            if (k < n) w[k] = wl[m * GT];
        }
    }
}

// Columns beyond kGivMax (linear_maxit > 255 without restarts): one thread.
__global__ void k_gmres_givens_serial(const double* __restrict__ part, GmresDev G, int j)
{
    const double s2 = sum_partials_warp(part, kMgsBlocks);
    if (threadIdx.x != 0) return;
    const double hnext = sqrt(s2);
    G.scal[1] = hnext;
    double* h = G.H + (long long)j * G.ld;
    h[j + 1] = hnext;
    for (int i = 0; i < j; ++i) {
        const double t = G.cs[i] * h[i] + G.sn[i] * h[i + 1];
        h[i + 1] = -G.sn[i] * h[i] + G.cs[i] * h[i + 1];
        h[i] = t;
    }
    const double r = hypot(h[j], hnext);
    if (r == 0.0) {
        *G.stop = 1;
        return;
    }
    G.cs[j] = h[j] / r;
    G.sn[j] = hnext / r;
    h[j] = r;
    G.g[j + 1] = -G.sn[j] * G.g[j];
    G.g[j] *= G.cs[j];
    const int m = j + 1;
    for (int i = m - 1; i >= 0; --i) {
        double s = G.g[i];
        for (int k2 = i + 1; k2 < m; ++k2) s -= G.H[(long long)k2 * G.ld + i] * G.y[k2];
        G.y[i] = s / G.H[(long long)i * G.ld + i];
    }
}

// Givens rotations of the new Hessenberg column and the back substitution
// R y = g (krylov.cpp:158-180), sequential in the reference's order on
// thread 0; the 1024-thread block stages every operand in shared memory first
// with coalesced loads (the column, rotations, g, and R in 32-row blocks), so
// the dependent chain runs on shared-memory latency instead of one L2 round
// trip per term (C3 at j ~ 67: 209 us -> ~10 us).
constexpr int kGivT = 1024, kGivRows = 16, kGivMax = 256;
__global__ void __launch_bounds__(kGivT) k_gmres_givens(const double* __restrict__ part, GmresDev G, int j)
{
    __shared__ double hs[kGivMax + 1], css[kGivMax], sns[kGivMax], gs[kGivMax + 1], ys[kGivMax];
    __shared__ double rb[kGivRows * kGivMax]; // R(i, k2) for a block of 32 rows i
    __shared__ int stop;
    const int t = threadIdx.x;
    const int m = j + 1;
    double* h = G.H + (long long)j * G.ld;
    for (int i = t; i < j + 1; i += kGivT) hs[i] = h[i];
    for (int i = t; i < j; i += kGivT) {
        css[i] = G.cs[i];
        sns[i] = G.sn[i];
    }
    for (int i = t; i <= j; i += kGivT) gs[i] = G.g[i];
    double s2 = 0.0;
    if (t < 32) s2 = sum_partials_warp(part, kMgsBlocks); // from the last k_mgs_dot
    __syncthreads();
    if (t == 0) {
        stop = 0;
        const double hnext = sqrt(s2);
        G.scal[1] = hnext;
        hs[j + 1] = hnext;
        for (int i = 0; i < j; ++i) {
            const double tt = css[i] * hs[i] + sns[i] * hs[i + 1];
            hs[i + 1] = -sns[i] * hs[i] + css[i] * hs[i + 1];
            hs[i] = tt;
        }
        const double r = hypot(hs[j], hnext);
        if (r == 0.0) {
            *G.stop = 1; // "gmres: zero pivot in Hessenberg triangularization"
            stop = 1;
        } else {
            const double c = hs[j] / r, sn = hnext / r;
            G.cs[j] = c;
            G.sn[j] = sn;
            hs[j] = r;
            gs[j + 1] = -sn * gs[j];
            gs[j] *= c;
            G.g[j + 1] = gs[j + 1];
            G.g[j] = gs[j];
        }
    }
    __syncthreads();
    for (int i = t; i <= j + 1; i += kGivT) h[i] = hs[i];
    if (stop) return;
    // back substitution in blocks of 32 rows, bottom up; row i needs
    // R(i, k2) = H[k2 * ld + i] for k2 > i (column k2 of the stored H)
    for (int i1 = m - 1; i1 >= 0; i1 -= kGivRows) {
        const int i0 = max(i1 - kGivRows + 1, 0);
        const int nr = i1 - i0 + 1;
        __syncthreads();
        for (int e = t; e < nr * m; e += kGivT) {
            const int k2 = e / nr, ii = e - k2 * nr; // consecutive threads: consecutive rows
            rb[ii * kGivMax + k2] = k2 == j ? hs[i0 + ii] : G.H[(long long)k2 * G.ld + i0 + ii];
        }
        __syncthreads();
        if (t == 0) {
            for (int i = i1; i >= i0; --i) {
                const double* row = rb + (i - i0) * kGivMax;
                double s = gs[i];
                for (int k2 = i + 1; k2 < m; ++k2) s -= row[k2] * ys[k2];
                ys[i] = s / row[i];
            }
        }
    }
    __syncthreads();
    for (int i = t; i < m; i += kGivT) G.y[i] = ys[i];
}

__global__ void k_relres(const double* __restrict__ part, const double* __restrict__ bnorm,
                         double* dst, const int* flags, const int* stop, double* status)
{
    const double s = sum_partials_warp(part, kRedBlocks);
    if (threadIdx.x == 0) {
        dst[0] = sqrt(s) / bnorm[0];
        if (status) { // the iteration's error flags and stop code next to the scalars:
            status[0] = (double)(flags ? flags[0] : 0); // one readback per Krylov iteration
            status[1] = (double)(stop ? stop[0] : 0);
        }
    }
}

// MINRES scalar slots
enum {
    kGamma = 0, kGammaPrev, kEta, kCPrev, kC, kSPrev, kS, kDelta, kGammaNext, kA0, kA1, kA2, kA3,
    kCNext, kSNext, kGammaSq, kGnSq
};

__global__ void k_minres_setup(const double* __restrict__ part, double* sc)
{
    const double s = sum_partials_warp(part, kRedBlocks);
    if (threadIdx.x != 0) return;
    sc[kGammaSq] = s;
    const double g = s > 0.0 ? sqrt(s) : 0.0;
    sc[kGamma] = g;
    sc[kGammaPrev] = 1.0;
    sc[kEta] = g;
    sc[kCPrev] = sc[kC] = 1.0;
    sc[kSPrev] = sc[kS] = 0.0;
}

__global__ void k_minres_delta(const double* __restrict__ part, double* sc)
{
    const double s = sum_partials_warp(part, kRedBlocks);
    if (threadIdx.x == 0) sc[kDelta] = s;
}

__global__ void k_minres_vnext(const double* __restrict__ az, const double* __restrict__ v,
                               const double* __restrict__ vprev, double* __restrict__ vnext,
                               const double* __restrict__ sc, int first, long long n)
{
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double c1 = -sc[kDelta] / sc[kGamma];
    double t = az[i] + c1 * v[i];
    if (!first) t = t + (-sc[kGamma] / sc[kGammaPrev]) * vprev[i];
    vnext[i] = t;
}

__global__ void k_minres_gamma(const double* __restrict__ part, double* sc, int* stop)
{
    const double gn_sq = sum_partials_warp(part, kRedBlocks);
    if (threadIdx.x != 0) return;
    sc[kGnSq] = gn_sq;
    if (gn_sq < 0.0) {
        *stop = 1; // "minres: preconditioner lost definiteness"
        return;
    }
    const double gn = sqrt(gn_sq);
    sc[kGammaNext] = gn;
    const double c = sc[kC], cp = sc[kCPrev], s = sc[kS], sp = sc[kSPrev];
    const double delta = sc[kDelta], gamma = sc[kGamma];
    const double a0 = c * delta - cp * s * gamma;
    const double a1 = sqrt(a0 * a0 + gn * gn);
    const double a2 = s * delta + cp * c * gamma;
    const double a3 = sp * gamma;
    sc[kA0] = a0;
    sc[kA1] = a1;
    sc[kA2] = a2;
    sc[kA3] = a3;
    if (a1 == 0.0) {
        *stop = 2;
        return;
    }
    sc[kCNext] = a0 / a1;
    sc[kSNext] = gn / a1;
}

__global__ void k_minres_update(const double* __restrict__ z, const double* __restrict__ wprev,
                                const double* __restrict__ w, double* __restrict__ wnext,
                                double* __restrict__ x, const double* __restrict__ sc,
                                const int* __restrict__ stop, long long n)
{
    if (*stop) return;
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double a1 = sc[kA1], a2 = sc[kA2], a3 = sc[kA3];
    double t = z[i] + (-a3) * wprev[i];
    t = t + (-a2) * w[i];
    t = t * (1.0 / a1);
    wnext[i] = t;
    x[i] += (sc[kCNext] * sc[kEta]) * t;
}

__global__ void k_minres_rotate(double* sc, const int* stop)
{
    if (*stop) return;
    sc[kEta] = -sc[kSNext] * sc[kEta];
    sc[kGammaPrev] = sc[kGamma];
    sc[kGamma] = sc[kGammaNext];
    sc[kCPrev] = sc[kC];
    sc[kC] = sc[kCNext];
    sc[kSPrev] = sc[kS];
    sc[kS] = sc[kSNext];
}

} // namespace

void launch_dot_partials(cudaStream_t s, const double* x, const double* y, long long n,
                         double* part)
{
    note_launch();
    k_dot_partials<<<kRedBlocks, kRedThreads, 0, s>>>(x, y, n, part);
}

void launch_finalize(cudaStream_t s, const double* part, double* dst, int mode)
{
    note_launch();
    k_finalize<<<1, 32, 0, s>>>(part, dst, mode);
}

void launch_copy(cudaStream_t s, const double* x, double* y, long long n)
{
    if (n > 0) { note_launch(); k_copy<<<blocks_for(n), kT, 0, s>>>(x, y, n); }
}

void launch_fill(cudaStream_t s, double* x, double v, long long n)
{
    if (n > 0) { note_launch(); k_fill<<<blocks_for(n), kT, 0, s>>>(x, v, n); }
}

void launch_scale_inv(cudaStream_t s, const double* x, const double* den, double* y, long long n,
                      const int* stop)
{
    note_launch();
    k_scale_inv<<<blocks_for(n), kT, 0, s>>>(x, den, y, n, stop);
}

void launch_axpy_neg(cudaStream_t s, const double* h, const double* v, double* w, long long n)
{
    note_launch();
    k_axpy_neg<<<blocks_for(n), kT, 0, s>>>(h, v, w, n);
}

void launch_combine(cudaStream_t s, const double* const* Ztab, const double* y, int m, double* x,
                    long long n, const double* xbase)
{
    note_launch();
    k_combine<<<blocks_for(n), kT, 0, s>>>(Ztab, y, m, x, n, xbase);
}

void launch_add(cudaStream_t s, const double* a, const double* b, double* out, long long n)
{
    note_launch();
    k_add<<<blocks_for(n), kT, 0, s>>>(a, b, out, n);
}

void launch_mgs_step(cudaStream_t s, const double* part, const GmresDev& G, int i, int j,
                     const double* vi, double* w, long long n)
{
    note_launch();
    k_mgs_step<<<kRedBlocks * 4, kT, 0, s>>>(part, G.H, G.ld, i, j, vi, w, n);
}

void launch_mgs_dot(cudaStream_t s, const double* part_in, const GmresDev& G, int i, int j,
                    const double* vi, double* w, const double* vnext, double* part_out, long long n)
{
    note_launch();
    k_mgs_dot<<<kMgsBlocks, kRedThreads, 0, s>>>(part_in, G.H, G.ld, i, j, vi, w, vnext, part_out, n);
}

void launch_dot_partials_mgs(cudaStream_t s, const double* x, const double* y, long long n,
                             double* part)
{
    note_launch();
    k_dot_partials<<<kMgsBlocks, kRedThreads, 0, s>>>(x, y, n, part);
}

std::atomic<int> g_mgs_persistent{8};

bool launch_mgs_persistent(cudaStream_t s, const double* const* V, double* w, const GmresDev& G,
                           int j, double* pa, double* pb, unsigned* bar, long long n)
{
    constexpr size_t smem = ((size_t)(kMgsBlocks / 148) * kMgsSmemM * 256 + kMgsBlocks) * sizeof(double);
    // one CTA per SM on a 148-SM B200, all co-resident; otherwise the caller
    // runs the launch-per-step sequence (same bits). Checked (and the shared
    // memory attribute set) once per device: 0 unknown, 1 usable, 2 not.
    static std::atomic<int> state[64];
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return false;
    int st = state[dev].load();
    if (st == 0) {
        st = [dev] {
        int sms = 0, per_sm = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms != 148 || kMgsBlocks % sms || (kMgsBlocks / sms) % (kMgsPersistThreads / 256)) return false;
        if (cudaFuncSetAttribute(k_mgs_persistent, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem) != cudaSuccess)
            return false;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_mgs_persistent, kMgsPersistThreads, smem);
        cudaGetLastError();
        return per_sm >= 1;
        }() ? 1 : 2;
        state[dev].store(st);
    }
    if (st != 1 || n > (long long)kMgsPersistM * kMgsBlocks * 256) return false;
    note_launch();
    double* H = G.H;
    int ld = G.ld;
    double* pfinal = (j & 1) ? pa : pb; // the natural output slot of step j
    void* args[] = {(void*)&V, (void*)&w, (void*)&H, (void*)&ld, (void*)&j,
                    (void*)&pa, (void*)&pb, (void*)&pfinal, (void*)&bar, (void*)&n};
    const cudaError_t e = cudaLaunchCooperativeKernel((const void*)k_mgs_persistent, dim3(148),
                                                      dim3(kMgsPersistThreads), args, smem, s);
    if (e != cudaSuccess) {
        // e.g. the SMs are shared with another context's kernels and the 148
        // CTAs cannot all be resident: fall back to the launch-per-step path
        cudaGetLastError();
        return false;
    }
    return true;
}

void launch_gmres_givens(cudaStream_t s, const double* part, const GmresDev& G, int j)
{
    note_launch();
    if (j + 1 >= kGivMax) k_gmres_givens_serial<<<1, 32, 0, s>>>(part, G, j);
    else k_gmres_givens<<<1, kGivT, 0, s>>>(part, G, j);
}

// |g_{j+1}| (the least-squares residual norm GMRES carries, = ||b - A x_j|| in exact
// arithmetic) with the error flags and stop code next to it, for the iterations
// whose true residual is not formed
__global__ void k_gmres_status(GmresDev G, int j, const int* flags, double* est, double* status)
{
    est[0] = fabs(G.g[j + 1]);
    status[0] = (double)(flags ? flags[0] : 0);
    status[1] = (double)G.stop[0];
}

std::atomic<int> g_gmres_lazy_residual{1};

void launch_gmres_status(cudaStream_t s, const GmresDev& G, int j, const int* flags, double* est,
                         double* status)
{
    note_launch();
    k_gmres_status<<<1, 1, 0, s>>>(G, j, flags, est, status);
}

void launch_relres(cudaStream_t s, const double* part, const double* bnorm, double* dst,
                   const int* flags, const int* stop, double* status)
{
    note_launch();
    k_relres<<<1, 32, 0, s>>>(part, bnorm, dst, flags, stop, status);
}

void launch_minres_setup(cudaStream_t s, const double* part, double* sc)
{
    note_launch();
    k_minres_setup<<<1, 32, 0, s>>>(part, sc);
}

void launch_minres_delta(cudaStream_t s, const double* part, double* sc)
{
    note_launch();
    k_minres_delta<<<1, 32, 0, s>>>(part, sc);
}

void launch_minres_vnext(cudaStream_t s, const double* az, const double* v, const double* vprev,
                         double* vnext, const double* sc, int first, long long n)
{
    note_launch();
    k_minres_vnext<<<blocks_for(n), kT, 0, s>>>(az, v, vprev, vnext, sc, first, n);
}

void launch_minres_gamma(cudaStream_t s, const double* part, double* sc, int* stop)
{
    note_launch();
    k_minres_gamma<<<1, 32, 0, s>>>(part, sc, stop);
}

void launch_minres_update(cudaStream_t s, const double* z, const double* wprev, const double* w,
                          double* wnext, double* x, const double* sc, const int* stop,
                          long long n)
{
    note_launch();
    k_minres_update<<<blocks_for(n), kT, 0, s>>>(z, wprev, w, wnext, x, sc, stop, n);
}

void launch_minres_rotate(cudaStream_t s, double* sc, const int* stop)
{
    note_launch();
    k_minres_rotate<<<1, 1, 0, s>>>(sc, stop);
}

} // namespace ocb
