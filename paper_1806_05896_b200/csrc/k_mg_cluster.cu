// Cluster-resident multigrid bottom solver (sm_100a, FP64).
//
// Levels <= 7 of a V-cycle are latency-bound: a level-7 colour pass touches
// 4K nodes, far too little work to amortise a kernel launch, and the
// reference's V-cycle runs 44 such dependent phases per level
// (multigrid.cpp:111-132). This kernel keeps the whole bottom of the
// hierarchy on chip in one thread-block cluster of kCS CTAs:
//   * "slab" levels (7 and 6): CTAs 1..kCS-1 each own a band of rows; their
//     x, b, r and the 9 coefficient arrays live in that CTA's shared memory.
//     A node on a band edge is also stored (remote DSM store) into the
//     neighbouring CTA's halo row as soon as it is updated, so every colour
//     pass reads only local shared memory; passes are separated by cluster
//     barriers (release/acquire makes the pushed halos visible);
//   * levels <= 5: CTA 0 alone holds everything in its shared memory and runs
//     with block barriers, then the 9x9 LU solve at level 2.
// Geometry is compile-time (template on the top level), so thread->node maps
// are shifts and masks. Semantics match the device V-cycle elsewhere: 4-colour
// symmetric Gauss-Seidel (forward 0..3 pre, backward 3..0 post), R = P^T,
// bilinear prolongation, zero coarse initial guesses and, when this kernel is
// the whole solve, `cycles` V-cycles with the ||r|| > 10 ||r_prev|| check of
// MgHierarchy::solve (multigrid.cpp:141-157).
#include "kernels.hpp"

#include <cooperative_groups.h>

#include <stdexcept>

namespace cg = cooperative_groups;

namespace ocb {

namespace {

constexpr int kCS = 16;          // CTAs per cluster (non-portable size)
constexpr int kW = kCS - 1;      // worker CTAs owning slab rows
constexpr int kCT = 1024;        // threads per CTA

template <int TOP>
struct Geo {
    static constexpr int NLEV = TOP - 1;                 // levels TOP..2
    static constexpr int nx(int k) { return (1 << (TOP - k)) - 1; }
    static constexpr bool slab(int k) { return nx(k) > 31; }
    static constexpr int rp(int k) { return (nx(k) + kW - 1) / kW; }
    static constexpr int cnt(int k) { return slab(k) ? rp(k) * nx(k) : nx(k) * nx(k); }
    // worker layout per slab level: coef 9*cnt, x, b, r, inv-diag (cnt each), halo above/below
    static constexpr int wsize(int k) { return 13 * cnt(k) + 2 * nx(k); }
    static constexpr int woff(int k) { return k == 0 ? 0 : woff(k - 1) + (slab(k - 1) ? wsize(k - 1) : 0); }
    // CTA-0 layout per coarse level: coef 9*cnt, x, b, inv-diag; one residual scratch at the end
    static constexpr int csize(int k) { return 12 * cnt(k); }
    // threads working a CTA-0 level: the colour lattice rounded up to whole warps
    static constexpr int c0threads(int k) { return ((((nx(k) + 1) / 2) * ((nx(k) + 1) / 2) + 31) / 32) * 32; }
    static constexpr int coff(int k) { return k == 0 ? 0 : coff(k - 1) + (slab(k - 1) ? 0 : csize(k - 1)); }
    static constexpr int first_c0() { return slab(0) ? (slab(1) ? 2 : 1) : 0; }
    static constexpr int cscratch() { return coff(NLEV - 1) + csize(NLEV - 1); }
    static constexpr int wtotal() { return woff(NLEV - 1) + (slab(NLEV - 1) ? wsize(NLEV - 1) : 0); }
    static constexpr int ctotal() { return cscratch() + cnt(first_c0()); }
    static constexpr int total() { return wtotal() > ctotal() ? wtotal() : ctotal(); }
};

// ------------------------------------------------------------ slab levels
template <int NX, int RP>
struct Slab {
    static constexpr int CNT = RP * NX;
    double* coef;   // [9][CNT]
    double* x;      // [CNT]
    double* b;
    double* r;
    double* inv;    // 1 / a_ii
    double* ha;     // halo row above (row r0-1), NX
    double* hb;     // halo row below (row r1), NX
    int w, r0, r1;  // worker index, own rows [r0, r1)

    __device__ Slab(double* base, unsigned rank)
    {
        coef = base;
        x = coef + 9 * CNT;
        b = x + CNT;
        r = b + CNT;
        inv = r + CNT;
        ha = inv + CNT;
        hb = ha + NX;
        w = (int)rank - 1;
        r0 = min(w * RP, NX); // trailing workers may own no rows
        r1 = min(r0 + RP, NX);
        if (w < 0) r0 = r1 = 0;
    }
    __device__ __forceinline__ double xat(int jx, int jy) const
    {
        if (jy < r0) return ha[jx];
        if (jy >= r1) return hb[jx];
        return x[(jy - r0) * NX + jx];
    }
};

// push an updated edge-row node into the neighbours' halos
template <int NX, int RP>
__device__ __forceinline__ void push_halo(cg::cluster_group& cl, const Slab<NX, RP>& s, int gx,
                                          int gy, double v, int base_off, double* smem)
{
    constexpr int HA = 13 * Slab<NX, RP>::CNT; // offset of ha in a slab
    if (gy == s.r0 && s.w > 0) {
        double* dst = cl.map_shared_rank(smem + base_off + HA + NX, (unsigned)s.w); // hb of w-1
        dst[gx] = v;
    }
    if (gy == s.r1 - 1 && s.r1 < NX) {
        double* dst = cl.map_shared_rank(smem + base_off + HA, (unsigned)(s.w + 2)); // ha of w+1
        dst[gx] = v;
    }
}

template <int NX, int RP>
__device__ void slab_sweep(cg::cluster_group& cl, const Slab<NX, RP>& s, bool forward, int off,
                           double* smem)
{
    constexpr int CNT = Slab<NX, RP>::CNT;
    for (int p = 0; p < 4; ++p) {
        const int col = forward ? p : 3 - p;
        const int cx = col & 1, cy = col >> 1;
        if (s.w >= 0) {
            const int y0 = s.r0 + (((s.r0 & 1) != cy) ? 1 : 0);
            const int gx = cx + 2 * (threadIdx.x & 63);
            const int gy = y0 + 2 * (threadIdx.x >> 6);
            if (gx < NX && gy < s.r1) {
                const int l = (gy - s.r0) * NX + gx;
                double acc = s.b[l];
#pragma unroll
                for (int d = 0; d < 9; ++d) {
                    if (d == 4) continue;
                    const int jx = gx + d % 3 - 1, jy = gy + d / 3 - 1;
                    if (jx < 0 || jx >= NX || jy < 0 || jy >= NX) continue;
                    acc -= s.coef[d * CNT + l] * s.xat(jx, jy);
                }
                const double v = acc * s.inv[l];
                s.x[l] = v;
                push_halo(cl, s, gx, gy, v, off, smem);
            }
        }
        cl.sync();
    }
}

template <int NX, int RP>
__device__ void slab_residual(const Slab<NX, RP>& s)
{
    constexpr int CNT = Slab<NX, RP>::CNT;
    if (s.w < 0) return;
    for (int idx = threadIdx.x; idx < CNT; idx += blockDim.x) {
        const int ly = idx / NX, gx = idx - ly * NX, gy = s.r0 + ly;
        if (gy >= s.r1) continue;
        double acc = 0.0;
#pragma unroll
        for (int d = 0; d < 9; ++d) {
            const int jx = gx + d % 3 - 1, jy = gy + d / 3 - 1;
            if (jx < 0 || jx >= NX || jy < 0 || jy >= NX) continue;
            acc += s.coef[d * CNT + idx] * s.xat(jx, jy);
        }
        s.r[idx] = s.b[idx] - acc;
    }
}

// ------------------------------------------------------------ CTA-0 levels
// Each CTA-0 level runs on the first T threads (its colour lattice rounded up to
// warps) and synchronises with a named barrier over exactly those threads, so
// the small levels do not pay a 32-warp __syncthreads per colour pass.
__device__ __forceinline__ void nbar(int id, int nthreads)
{
    if (nthreads <= 32) __syncwarp();
    else asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

template <int NX, int T, int BAR>
__device__ void c0_sweep(const double* coef, double* x, const double* b, const double* inv,
                         bool forward)
{
    constexpr int N = NX * NX;
    constexpr int LX = (NX + 1) / 2;
    for (int p = 0; p < 4; ++p) {
        const int col = forward ? p : 3 - p;
        const int cx = col & 1, cy = col >> 1;
        const int gx = cx + 2 * (threadIdx.x % LX), gy = cy + 2 * (threadIdx.x / LX);
        if (gx < NX && gy < NX) {
            const int i = gy * NX + gx;
            double acc = b[i];
#pragma unroll
            for (int d = 0; d < 9; ++d) {
                if (d == 4) continue;
                const int jx = gx + d % 3 - 1, jy = gy + d / 3 - 1;
                if (jx < 0 || jx >= NX || jy < 0 || jy >= NX) continue;
                acc -= coef[d * N + i] * x[jy * NX + jx];
            }
            x[i] = acc * inv[i];
        }
        nbar(BAR, T);
    }
}

template <int NX, int T, int BAR>
__device__ void c0_residual(const double* coef, const double* x, const double* b, double* r)
{
    constexpr int N = NX * NX;
    for (int i = threadIdx.x; i < N; i += T) {
        const int gy = i / NX, gx = i - gy * NX;
        double acc = 0.0;
#pragma unroll
        for (int d = 0; d < 9; ++d) {
            const int jx = gx + d % 3 - 1, jy = gy + d / 3 - 1;
            if (jx < 0 || jx >= NX || jy < 0 || jy >= NX) continue;
            acc += coef[d * N + i] * x[jy * NX + jx];
        }
        r[i] = b[i] - acc;
    }
    nbar(BAR, T);
}

// R = P^T restriction from a fine residual accessor
template <typename F>
__device__ __forceinline__ double restrict_from(const F& fr, int cx, int cy)
{
    double s = 0.0;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const double wy = (a == 1) ? 1.0 : 0.5;
#pragma unroll
        for (int b = 0; b < 3; ++b) {
            const double wx = (b == 1) ? 1.0 : 0.5;
            s += (wx * wy) * fr(2 * cx + b, 2 * cy + a);
        }
    }
    return s;
}

// bilinear prolongation value at fine (gx, gy) from a coarse accessor (NXC per side)
template <int NXC, typename F>
__device__ __forceinline__ double prolong_from(const F& cxv, int gx, int gy)
{
    int px[2], py[2];
    double wx[2], wy[2];
    int nxn = 0, nyn = 0;
    if (gx & 1) { px[0] = (gx - 1) >> 1; wx[0] = 1.0; nxn = 1; }
    else {
        if (gx / 2 - 1 >= 0) { px[nxn] = gx / 2 - 1; wx[nxn++] = 0.5; }
        if (gx / 2 < NXC) { px[nxn] = gx / 2; wx[nxn++] = 0.5; }
    }
    if (gy & 1) { py[0] = (gy - 1) >> 1; wy[0] = 1.0; nyn = 1; }
    else {
        if (gy / 2 - 1 >= 0) { py[nyn] = gy / 2 - 1; wy[nyn++] = 0.5; }
        if (gy / 2 < NXC) { py[nyn] = gy / 2; wy[nyn++] = 0.5; }
    }
    double e = 0.0;
    for (int a = 0; a < nyn; ++a)
        for (int b = 0; b < nxn; ++b) e += (wx[b] * wy[a]) * cxv(px[b], py[a]);
    return e;
}

// load a level operator (materialising constant stencil + diag) rows [r0, r1)
// into 9 coefficient arrays plus the reciprocal diagonal used by the smoother
__device__ void load_op(const Op9& A, int nx, int r0, int r1, int cnt, double* coef, double* inv)
{
    const long long n = (long long)nx * nx;
    for (int idx = threadIdx.x; idx < (r1 - r0) * nx; idx += blockDim.x) {
        const long long gi = (long long)r0 * nx + idx;
#pragma unroll
        for (int d = 0; d < 9; ++d) {
            double v = A.coef ? __ldg(A.coef + d * n + gi) : A.c[d];
            if (d == 4 && A.diag) v += __ldg(A.diag + gi);
            coef[d * cnt + idx] = v;
            if (d == 4) inv[idx] = 1.0 / v;
        }
    }
}

// CTA-0 part of the V-cycle for levels K..NLEV-1 (all <= 31 per side). Runs on
// threads [0, T_K); callers keep the other threads out.
template <int TOP, int K>
struct C0Down {
    using G = Geo<TOP>;
    static __device__ void run(double* smem, const BottomArgs& a, int pre, int post)
    {
        constexpr int NX = G::nx(K);
        constexpr int N = NX * NX;
        constexpr int T = G::c0threads(K);
        constexpr int BAR = 1 + K; // named barrier per level (0 is __syncthreads)
        double* coef = smem + G::coff(K);
        double* x = coef + 9 * N;
        double* b = x + N;
        double* inv = b + N;
        if constexpr (K == G::NLEV - 1) {
            // level 2: dense 9x9 LU solve (DenseFactor::solve)
            if (threadIdx.x == 0) {
                double y[9];
                for (int i = 0; i < 9; ++i) y[i] = b[a.perm[i]];
                for (int i = 0; i < 9; ++i)
                    for (int k2 = 0; k2 < i; ++k2) y[i] -= a.lu[k2 * 9 + i] * y[k2];
                for (int i = 8; i >= 0; --i) {
                    for (int k2 = i + 1; k2 < 9; ++k2) y[i] -= a.lu[k2 * 9 + i] * y[k2];
                    y[i] /= a.lu[i * 9 + i];
                }
                for (int i = 0; i < 9; ++i) x[i] = y[i];
            }
            __syncwarp();
        } else {
            constexpr int NC = G::nx(K + 1);
            constexpr int TC = G::c0threads(K + 1);
            double* r = smem + G::cscratch();
            double* cb = smem + G::coff(K + 1) + 10 * NC * NC;
            double* cx = smem + G::coff(K + 1) + 9 * NC * NC;
            for (int s = 0; s < pre; ++s) c0_sweep<NX, T, BAR>(coef, x, b, inv, true);
            c0_residual<NX, T, BAR>(coef, x, b, r);
            for (int I = threadIdx.x; I < NC * NC; I += T) {
                const int cy = I / NC, cxx = I - cy * NC;
                cb[I] = restrict_from([&](int gx, int gy) { return r[gy * NX + gx]; }, cxx, cy);
                cx[I] = 0.0;
            }
            nbar(BAR, T);
            if (threadIdx.x < TC) C0Down<TOP, K + 1>::run(smem, a, pre, post);
            nbar(BAR, T);
            for (int i = threadIdx.x; i < N; i += T) {
                const int gy = i / NX, gx = i - gy * NX;
                x[i] = x[i] + prolong_from<NC>([&](int u, int v) { return cx[v * NC + u]; }, gx, gy);
            }
            nbar(BAR, T);
            for (int s = 0; s < post; ++s) c0_sweep<NX, T, BAR>(coef, x, b, inv, false);
        }
    }
};

// --------------------------------------------------------------- kernel
// Optional phase timestamps (%globaltimer) of CTAs 0 and 1 for tuning.
__device__ int g_probe_on = 0;
__device__ unsigned long long g_tprobe[64];
__device__ __forceinline__ void probe(unsigned rank, int i)
{
    if (threadIdx.x == 0 && rank < 2 && g_probe_on) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g_tprobe[rank * 32 + i] = t;
    }
}

template <int TOP>
__global__ void __launch_bounds__(kCT, 1)
    k_bottom_cluster(BottomArgs a, const double* __restrict__ bg, double* __restrict__ xg,
                     int cycles, int pre, int post, int check, double* state, int* flags)
{
    using G = Geo<TOP>;
    constexpr int NX0 = G::nx(0), RP0 = G::rp(0);
    constexpr int NX1 = G::nx(1), RP1 = G::rp(1);
    constexpr bool S1 = G::slab(1); // TOP = 7: levels 7 and 6 are slab levels
    constexpr int OFF1 = G::woff(1);
    constexpr int C0 = G::first_c0();
    extern __shared__ double smem[];
    __shared__ double red[64];
    cg::cluster_group cl = cg::this_cluster();
    const unsigned rank = cl.block_rank();
    probe(rank, 0);

    Slab<NX0, RP0> s0(smem + G::woff(0), rank);
    Slab<NX1, RP1> s1(smem + OFF1, rank); // only meaningful when S1

    // ---- load operators and the top-level rhs
    if (rank != 0) {
        load_op(a.ops[0], NX0, s0.r0, s0.r1, Slab<NX0, RP0>::CNT, s0.coef, s0.inv);
        for (int idx = threadIdx.x; idx < (s0.r1 - s0.r0) * NX0; idx += blockDim.x) {
            s0.x[idx] = 0.0;
            s0.b[idx] = bg[(long long)s0.r0 * NX0 + idx];
        }
        for (int i = threadIdx.x; i < 2 * NX0; i += blockDim.x) s0.ha[i] = 0.0; // ha, hb contiguous
        if constexpr (S1)
            load_op(a.ops[1], NX1, s1.r0, s1.r1, Slab<NX1, RP1>::CNT, s1.coef, s1.inv);
    } else {
        for (int k = C0; k < G::NLEV; ++k) {
            const int nx = (1 << (TOP - k)) - 1;
            double* base = smem + G::coff(k);
            load_op(a.ops[k], nx, 0, nx, nx * nx, base, base + 11 * nx * nx);
        }
    }
    cl.sync();
    probe(rank, 1);

    auto top_norm = [&](const double* v) -> double {
        double acc = 0.0;
        if (rank != 0)
            for (int idx = threadIdx.x; idx < (s0.r1 - s0.r0) * NX0; idx += blockDim.x)
                acc += v[idx] * v[idx];
        acc = block_sum(acc, red);
        if (threadIdx.x == 0) {
            double* dst = cl.map_shared_rank(&red[34], 0);
            dst[rank] = acc;
        }
        cl.sync();
        double tot = 0.0;
        if (rank == 0 && threadIdx.x == 0)
            for (int q = 0; q < kCS; ++q) tot += red[34 + q];
        cl.sync();
        return sqrt(tot);
    };
    double prev = 0.0;
    if (check) prev = top_norm(s0.b);

    for (int cyc = 0; cyc < cycles; ++cyc) {
        // ===================== level 0 (slab) down
        for (int s = 0; s < pre; ++s) slab_sweep<NX0, RP0>(cl, s0, true, G::woff(0), smem);
        probe(rank, 2);
        slab_residual<NX0, RP0>(s0);
        cl.sync();
        probe(rank, 3);
        if constexpr (S1) {
            // restrict into the level-1 slab rows this CTA owns (fine rows may be remote)
            if (rank != 0) {
                auto fr = [&](int gx, int gy) -> double {
                    const int owner = gy / RP0 + 1;
                    const double* rr = (owner == (int)rank)
                                           ? s0.r
                                           : cl.map_shared_rank(s0.r, (unsigned)owner);
                    return rr[(gy - (owner - 1) * RP0) * NX0 + gx];
                };
                for (int idx = threadIdx.x; idx < (s1.r1 - s1.r0) * NX1; idx += blockDim.x) {
                    const int ly = idx / NX1, cx = idx - ly * NX1;
                    s1.b[idx] = restrict_from(fr, cx, s1.r0 + ly);
                    s1.x[idx] = 0.0;
                }
                for (int i = threadIdx.x; i < 2 * NX1; i += blockDim.x) s1.ha[i] = 0.0;
            }
            cl.sync();
            probe(rank, 4);
            // ===================== level 1 (slab) down
            for (int s = 0; s < pre; ++s) slab_sweep<NX1, RP1>(cl, s1, true, OFF1, smem);
            probe(rank, 5);
            slab_residual<NX1, RP1>(s1);
            cl.sync();
            probe(rank, 6);
        }
        // restrict the last slab level into CTA 0's first coarse level
        constexpr int NLS = S1 ? NX1 : NX0; // last slab level size
        constexpr int RPLS = S1 ? RP1 : RP0;
        constexpr int NC = G::nx(C0);
        if (rank == 0) {
            const double* rloc = S1 ? s1.r : s0.r;
            double* cb = smem + G::coff(C0) + 10 * NC * NC;
            double* cxv = smem + G::coff(C0) + 9 * NC * NC;
            auto fr = [&](int gx, int gy) -> double {
                const int owner = gy / RPLS + 1;
                const double* rr = cl.map_shared_rank(rloc, (unsigned)owner);
                return rr[(gy - (owner - 1) * RPLS) * NLS + gx];
            };
            for (int I = threadIdx.x; I < NC * NC; I += blockDim.x) {
                const int cy = I / NC, cxx = I - cy * NC;
                cb[I] = restrict_from(fr, cxx, cy);
                cxv[I] = 0.0;
            }
            __syncthreads();
            probe(rank, 7);
            // ===================== CTA-0 levels (<= 31 per side) and the LU solve
            if (threadIdx.x < G::c0threads(C0)) C0Down<TOP, C0>::run(smem, a, pre, post);
            probe(rank, 8);
        }
        cl.sync();
        probe(rank, 9);
        // ===================== prolongate CTA 0's correction into the last slab level
        {
            const double* c0x = cl.map_shared_rank(smem + G::coff(C0) + 9 * NC * NC, 0);
            auto cxv = [&](int u, int v) { return c0x[v * NC + u]; };
            if constexpr (S1) {
                if (rank != 0)
                    for (int idx = threadIdx.x; idx < (s1.r1 - s1.r0) * NX1; idx += blockDim.x) {
                        const int ly = idx / NX1, gx = idx - ly * NX1, gy = s1.r0 + ly;
                        const double v = s1.x[idx] + prolong_from<NC>(cxv, gx, gy);
                        s1.x[idx] = v;
                        push_halo(cl, s1, gx, gy, v, OFF1, smem);
                    }
                cl.sync();
                probe(rank, 10);
                for (int s = 0; s < post; ++s) slab_sweep<NX1, RP1>(cl, s1, false, OFF1, smem);
                probe(rank, 11);
                // prolongate level 1 into level 0 (coarse rows may be remote)
                if (rank != 0) {
                    auto c1x = [&](int u, int v) -> double {
                        const int owner = v / RP1 + 1;
                        const double* xx = (owner == (int)rank)
                                               ? s1.x
                                               : cl.map_shared_rank(s1.x, (unsigned)owner);
                        return xx[(v - (owner - 1) * RP1) * NX1 + u];
                    };
                    for (int idx = threadIdx.x; idx < (s0.r1 - s0.r0) * NX0; idx += blockDim.x) {
                        const int ly = idx / NX0, gx = idx - ly * NX0, gy = s0.r0 + ly;
                        const double v = s0.x[idx] + prolong_from<NX1>(c1x, gx, gy);
                        s0.x[idx] = v;
                        push_halo(cl, s0, gx, gy, v, G::woff(0), smem);
                    }
                }
            } else {
                if (rank != 0)
                    for (int idx = threadIdx.x; idx < (s0.r1 - s0.r0) * NX0; idx += blockDim.x) {
                        const int ly = idx / NX0, gx = idx - ly * NX0, gy = s0.r0 + ly;
                        const double v = s0.x[idx] + prolong_from<NC>(cxv, gx, gy);
                        s0.x[idx] = v;
                        push_halo(cl, s0, gx, gy, v, G::woff(0), smem);
                    }
            }
            cl.sync();
            probe(rank, 12);
        }
        for (int s = 0; s < post; ++s) slab_sweep<NX0, RP0>(cl, s0, false, G::woff(0), smem);
        probe(rank, 13);
        if (check) {
            slab_residual<NX0, RP0>(s0);
            __syncthreads();
            const double res = top_norm(s0.r);
            if (rank == 0 && threadIdx.x == 0 && res > 10.0 * prev) atomicOr(flags, kErrMgDiverged);
            prev = res;
        }
    }
    if (rank != 0)
        for (int idx = threadIdx.x; idx < (s0.r1 - s0.r0) * NX0; idx += blockDim.x)
            xg[(long long)s0.r0 * NX0 + idx] = s0.x[idx];
    if (check && state && rank == 0 && threadIdx.x == 0) state[0] = prev;
}

template <int TOP>
void launch_top(cudaStream_t s, const BottomArgs& a, const double* b, double* x, int cycles,
                int pre, int post, bool check, double* state, int* flags)
{
    const size_t smem = (size_t)Geo<TOP>::total() * sizeof(double);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_bottom_cluster<TOP>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        cudaFuncSetAttribute(k_bottom_cluster<TOP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
        attr = true;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(kCS);
    cfg.blockDim = dim3(kCT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at{};
    at.id = cudaLaunchAttributeClusterDimension;
    at.val.clusterDim.x = kCS;
    at.val.clusterDim.y = 1;
    at.val.clusterDim.z = 1;
    cfg.attrs = &at;
    cfg.numAttrs = 1;
    note_launch();
    cudaLaunchKernelEx(&cfg, k_bottom_cluster<TOP>, a, b, x, cycles, pre, post, check ? 1 : 0,
                       state, flags);
}

static_assert(Geo<7>::total() * 8 <= 220 * 1024, "level-7 cluster layout exceeds shared memory");

} // namespace

void cluster_probes(int enable, unsigned long long* out64)
{
    cudaMemcpyToSymbol(g_probe_on, &enable, sizeof(int));
    if (out64) cudaMemcpyFromSymbol(out64, g_tprobe, 64 * sizeof(unsigned long long));
}

bool cluster_bottom_supported()
{
    static int supported = -1;
    if (supported < 0) {
        supported = 0;
        const size_t smem = (size_t)Geo<7>::total() * sizeof(double);
        if (cudaFuncSetAttribute(k_bottom_cluster<7>,
                                 cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess &&
            cudaFuncSetAttribute(k_bottom_cluster<7>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem) == cudaSuccess) {
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3(kCS);
            cfg.blockDim = dim3(kCT);
            cfg.dynamicSmemBytes = smem;
            cudaLaunchAttribute at{};
            at.id = cudaLaunchAttributeClusterDimension;
            at.val.clusterDim.x = kCS;
            at.val.clusterDim.y = 1;
            at.val.clusterDim.z = 1;
            cfg.attrs = &at;
            cfg.numAttrs = 1;
            int nclusters = 0;
            if (cudaOccupancyMaxActiveClusters(&nclusters, k_bottom_cluster<7>, &cfg) == cudaSuccess &&
                nclusters > 0)
                supported = 1;
        }
        cudaGetLastError();
    }
    return supported == 1;
}

void launch_bottom_cluster(cudaStream_t s, const ClusterArgs& a, const double* b, double* x,
                           int cycles, int pre, int post, bool check, double* state, int* flags)
{
    if (a.ops[0].nx == 127) launch_top<7>(s, a, b, x, cycles, pre, post, check, state, flags);
    else if (a.ops[0].nx == 63) launch_top<6>(s, a, b, x, cycles, pre, post, check, state, flags);
    else throw std::runtime_error("cluster bottom: top level must be 6 or 7");
}

} // namespace ocb
