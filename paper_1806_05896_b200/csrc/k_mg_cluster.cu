// Cluster-resident multigrid bottom solver (sm_100a, FP64).
//
// Levels <= 7 of a V-cycle are latency-bound: a level-7 colour pass touches
// 4K nodes, far too little work to amortise a kernel launch, and the
// reference's V-cycle runs 44 dependent phases per level
// (multigrid.cpp:111-132). This kernel keeps the bottom of the hierarchy on
// chip in one thread-block cluster of 16 CTAs x 256 threads:
//   * slab levels (the top level TOP = 7 or 6, and level 6 below a level-7
//     top): CTA w owns rows [RP*w, RP*w+RP). Thread t owns one node of EACH
//     colour (same position in the four colour sub-grids), so every colour
//     pass keeps all warps busy and no warp burns issue slots idling; the top
//     level keeps the 4 nodes' 9 coefficients, 1/a_ii and b in registers.
//     x is stored colour-planar with one halo row above and below, so every
//     neighbour read is a conflict-free shared-memory load.
//   * halo exchange is dataflow, not a cluster barrier: after a colour pass a
//     band-edge node st.async's its new value into the neighbour CTA's halo
//     row, completing bytes on that CTA's per-colour mbarrier; a CTA waits on
//     its mbarrier only before a pass that reads that colour of a halo row.
//     (Only the first band row, colours 0/1, feeds the CTA above; only the
//     last, colours 2/3, feeds the CTA below.) Prolongation of halo rows is
//     recomputed locally from the same parents (bit-identical), so there are
//     no exchange events outside the smoothing passes;
//   * levels <= 5 run in CTA 0 alone (planar shared memory, block barriers),
//     ending with the 9x9 LU solve at level 2 (factor held in shared memory).
// Semantics match the tiled V-cycle levels: 4-colour symmetric Gauss-Seidel
// (forward colours 0..3 pre, backward 3..0 post), R = P^T restriction of the
// residual, bilinear prolongation, zero coarse initial guesses and, when this
// kernel is the whole solve, `cycles` V-cycles with the ||r|| > 10 ||r_prev||
// check of MgHierarchy::solve (multigrid.cpp:141-157).
#include "kernels.hpp"

#include <cooperative_groups.h>

#include <cstdint>
#include <stdexcept>

namespace cg = cooperative_groups;

namespace ocb {

namespace {

constexpr int kCS = 16;  // CTAs per cluster (non-portable size)
constexpr int kCT = 256; // threads per CTA

// --------------------------------------------------- mbarrier / DSM primitives
__device__ __forceinline__ uint32_t saddr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t rank)
{
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
    return r;
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect(uint32_t bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity)
{
    uint32_t done = 0;
    while (!done) {
        asm volatile("{\n .reg .pred p;\n"
                     " mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n"
                     " selp.u32 %0, 1, 0, p;\n}"
                     : "=r"(done)
                     : "r"(bar), "r"(parity)
                     : "memory");
    }
}

__device__ __forceinline__ void st_async(uint32_t raddr, double v, uint32_t rbar)
{
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(raddr),
                 "l"(__double_as_longlong(v)), "r"(rbar)
                 : "memory");
}

// ------------------------------------------------------------- geometry
__host__ __device__ constexpr int fl2(int v) { return (v - (((v % 2) + 2) % 2)) / 2; } // floor(v / 2)

// Colour-planar layouts: plane (gx & 1) + 2 (row & 1) holds the nodes of one
// colour; rows of a plane are padded by one leading column (and the CTA-0
// levels by one leading row) that stay zero, so a neighbour outside the
// domain reads 0 and every neighbour of a thread's colour-c node is
// x[q + nb(c, dx, dy)] with a compile-time offset and q = rr * SX + cc.
template <int NX_, int RP_>
struct SlabG {
    static constexpr int NX = NX_, RP = RP_;
    static constexpr int WX = (NX + 1) / 2;     // columns per colour row
    static constexpr int SX = WX + 1;           // padded row stride
    static constexpr int RH = RP / 2;           // colour rows per band
    static constexpr int PS = (RH + 1) * SX;    // plane size (incl. the halo rows)
    static constexpr int XS = 4 * PS;           // planar x with halos
    static constexpr int GROUP = RH * WX;       // threads owning nodes (one per colour)
    static constexpr int RS = RP * NX;          // row-major residual of own rows
    static_assert(RP % 2 == 0, "even row bands keep the colour parity per CTA");
    static_assert(GROUP <= kCT, "one node per colour per thread");
    static_assert(2 * NX <= kCT, "one halo node per thread");
    // planar index of (gx, local row lr); lr = gy - r0 + 1 in [0, RP + 1]
    __host__ __device__ static constexpr int xi(int gx, int lr)
    {
        return ((gx & 1) + 2 * (lr & 1)) * PS + (lr >> 1) * SX + fl2(gx) + 1;
    }
    // offset of neighbour (dx, dy) of the colour-c node at (cc, rr), relative to q
    __host__ __device__ static constexpr int nb(int c, int dx, int dy)
    {
        return xi((c & 1) + dx, (c >> 1) + 1 + dy);
    }
    // bytes of one colour segment of a row (colours 0, 2: even gx; 1, 3: odd gx)
    __device__ static __forceinline__ uint32_t seg_bytes(int c) { return 8u * ((c & 1) ? NX / 2 : (NX + 1) / 2); }
};

template <int NX>
struct FullG { // CTA-0 level: planar x, b, inv, r, coefficients; padded, no halos
    static constexpr int WX = (NX + 1) / 2;
    static constexpr int SX = WX + 1;
    static constexpr int PS = (WX + 1) * SX;
    static constexpr int S = 4 * PS;
    static_assert(WX * WX <= kCT, "one node per colour per thread");
    __host__ __device__ static constexpr int xi(int gx, int gy)
    {
        return ((gx & 1) + 2 * (gy & 1)) * PS + (fl2(gy) + 1) * SX + fl2(gx) + 1;
    }
    __host__ __device__ static constexpr int nb(int c, int dx, int dy) { return xi((c & 1) + dx, (c >> 1) + dy); }
};

// The four nodes (one per colour c) a thread owns on a slab level:
// gx = 2 cc + (c & 1), gy = r0 + 2 rr + (c >> 1), local row lr = gy - r0 + 1.
template <class G>
struct Own {
    int cc, rr, r0, q;
    bool thr; // thread owns nodes on this level
    __device__ explicit Own(int w)
    {
        const int t = threadIdx.x;
        thr = t < G::GROUP;
        rr = t / G::WX;
        cc = t - rr * G::WX;
        r0 = G::RP * w;
        q = rr * G::SX + cc;
    }
    __device__ __forceinline__ int gx(int c) const { return 2 * cc + (c & 1); }
    __device__ __forceinline__ int gy(int c) const { return r0 + 2 * rr + (c >> 1); }
    __device__ __forceinline__ int lr(int c) const { return 2 * rr + (c >> 1) + 1; }
    __device__ __forceinline__ bool valid(int c) const { return thr && gx(c) < G::NX && gy(c) < G::NX; }
    __device__ __forceinline__ int me(int c) const { return q + G::nb(c, 0, 0); }
    __device__ __forceinline__ int slot(int c) const { return c * G::GROUP + threadIdx.x; }
};

// x(gx+dx, gy+dy) of the colour-c node from the local planar band (own rows +
// halo rows; outside the domain the zero padding / never-written slots read 0)
template <class G>
__device__ __forceinline__ double xnb(const double* xs, const Own<G>& o, int c, int dx, int dy)
{
    return xs[o.q + G::nb(c, dx, dy)];
}

// Halo exchange state of one slab level. mbarrier c of a CTA counts the bytes
// of colour c arriving in its halo rows: colours 0/1 from the CTA below (its
// first row), colours 2/3 from the CTA above (its last row). Bit c of `pend`
// marks an exchange of colour c not yet consumed, bit c of `par` the parity of
// the next phase of barrier c. At most one exchange per colour is ever in
// flight: a neighbour's next colour-c pass depends on values this CTA sends
// only after consuming the previous one (and every V-cycle phase boundary
// consumes all exchanges), so parity waits cannot alias.
template <class G>
struct Halo {
    uint32_t bar; // local mbarriers (4 x 8 bytes)
    uint32_t xs;  // local planar x (shared address)
    int w;
    unsigned pend, par;

    __device__ void setup(uint64_t* bars, double* x, int rank)
    {
        bar = saddr(bars);
        xs = saddr(x);
        w = rank;
        pend = par = 0u;
    }
    __device__ bool has_up() const { return w > 0; }
    __device__ bool has_dn() const { return G::RP * (w + 1) < G::NX; }
    // thread 0: init and arm phase 0 of the four barriers
    __device__ void init_barriers() const
    {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            mbar_init(bar + 8 * c, 1);
            mbar_expect(bar + 8 * c, G::seg_bytes(c));
        }
    }
    __device__ __forceinline__ void ensure(int c)
    {
        if (!((pend >> c) & 1u)) return;
        pend &= ~(1u << c);
        if (!(c < 2 ? has_dn() : has_up())) return;
        mbar_wait(bar + 8 * c, (par >> c) & 1u);
        par ^= 1u << c;
        if (threadIdx.x == 0) mbar_expect(bar + 8 * c, G::seg_bytes(c));
    }
    __device__ __forceinline__ void ensure_all()
    {
#pragma unroll
        for (int c = 0; c < 4; ++c) ensure(c);
    }
    // after the CTA barrier of a colour-c pass: send the band-edge value
    __device__ __forceinline__ void push(const Own<G>& o, double v, int c) const
    {
        if (c < 2 && o.rr == 0 && has_up())
            st_async(mapa(xs + 8u * G::xi(o.gx(c), G::RP + 1), (uint32_t)(w - 1)), v,
                     mapa(bar + 8 * c, (uint32_t)(w - 1)));
        if (c >= 2 && o.rr == G::RH - 1 && has_dn())
            st_async(mapa(xs + 8u * G::xi(o.gx(c), 0), (uint32_t)(w + 1)), v,
                     mapa(bar + 8 * c, (uint32_t)(w + 1)));
    }
    __device__ __forceinline__ void passed(int c) { pend |= 1u << c; }
};

// One symmetric-colour GS sweep on a slab level. upd(c) returns the new value
// of the thread's colour-c node.
template <bool FWD, class G, typename U>
__device__ __forceinline__ void slab_sweep(double* xs, Halo<G>& H, const Own<G>& o, const U& upd)
{
#pragma unroll
    for (int p = 0; p < 4; ++p) {
        const int c = FWD ? p : 3 - p;
        if (c < 2) { // first-row nodes read the upper halo (colours 2, 3)
            H.ensure(2);
            H.ensure(3);
        } else { // last-row nodes read the lower halo (colours 0, 1)
            H.ensure(0);
            H.ensure(1);
        }
        const bool act = o.valid(c);
        double v = 0.0;
        if (act) {
            v = upd(c);
            xs[o.me(c)] = v;
        }
        __syncthreads(); // CTA-local visibility; every halo read of this pass is done
        if (act) H.push(o, v, c);
        H.passed(c);
    }
}

// ----------------------------------------------------------- CTA-0 levels
template <int NX>
struct C0Level {
    double* coef; // [9][S] planar
    double* x;    // [S]
    double* b;
    double* inv;
    double* r;
};

template <bool FWD, int NX>
__device__ __forceinline__ void c0_sweep(const C0Level<NX>& L)
{
    using G = FullG<NX>;
    const int t = threadIdx.x;
    const int rr = t / G::WX, cc = t - rr * G::WX;
    const int q = rr * G::SX + cc;
    const bool thr = t < G::WX * G::WX;
#pragma unroll
    for (int p = 0; p < 4; ++p) {
        const int c = FWD ? p : 3 - p;
        const int gx = 2 * cc + (c & 1), gy = 2 * rr + (c >> 1);
        if (thr && gx < NX && gy < NX) {
            const int me = q + G::nb(c, 0, 0);
            double s = L.b[me];
#pragma unroll
            for (int d = 0; d < 9; ++d) {
                if (d == 4) continue;
                s -= L.coef[d * G::S + me] * L.x[q + G::nb(c, d % 3 - 1, d / 3 - 1)];
            }
            L.x[me] = s * L.inv[me];
        }
        __syncthreads();
    }
}

template <int NX>
__device__ __forceinline__ void c0_residual(const C0Level<NX>& L)
{
    using G = FullG<NX>;
    for (int i = threadIdx.x; i < NX * NX; i += blockDim.x) {
        const int gy = i / NX, gx = i - gy * NX;
        const int me = G::xi(gx, gy);
        double s = 0.0;
#pragma unroll
        for (int d = 0; d < 9; ++d) {
            const int jx = gx + d % 3 - 1, jy = gy + d / 3 - 1;
            if (jx < 0 || jx >= NX || jy < 0 || jy >= NX) continue;
            s += L.coef[d * G::S + me] * L.x[G::xi(jx, jy)];
        }
        L.r[me] = L.b[me] - s;
    }
    __syncthreads();
}

// (R r)(cx, cy) with R = P^T: fine nodes 2c, 2c+1, 2c+2 weighted 1/2, 1, 1/2 per axis
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

// parents of fine index g on one axis: (i0, w0), (i1, w1); weight 0 = absent
template <int NXC>
__device__ __forceinline__ void parents(int g, int& i0, int& i1, double& w0, double& w1)
{
    if (g & 1) {
        i0 = i1 = (g - 1) >> 1;
        w0 = 1.0;
        w1 = 0.0;
    } else {
        i0 = g / 2 - 1;
        i1 = g / 2;
        w0 = i0 >= 0 ? 0.5 : 0.0;
        w1 = i1 < NXC ? 0.5 : 0.0;
    }
}

// (P e)(gx, gy): bilinear interpolation from the coarse level of size NXC
template <int NXC, typename F>
__device__ __forceinline__ double prolong_from(const F& cxv, int gx, int gy)
{
    int x0, x1, y0, y1;
    double wx0, wx1, wy0, wy1;
    parents<NXC>(gx, x0, x1, wx0, wx1);
    parents<NXC>(gy, y0, y1, wy0, wy1);
    double e = 0.0;
    if (wy0 != 0.0) {
        if (wx0 != 0.0) e += (wx0 * wy0) * cxv(x0, y0);
        if (wx1 != 0.0) e += (wx1 * wy0) * cxv(x1, y0);
    }
    if (wy1 != 0.0) {
        if (wx0 != 0.0) e += (wx0 * wy1) * cxv(x0, y1);
        if (wx1 != 0.0) e += (wx1 * wy1) * cxv(x1, y1);
    }
    return e;
}

__device__ __forceinline__ double op_entry(const Op9& A, int d, long long n, long long i)
{
    double v = A.coef ? __ldg(A.coef + d * n + i) : A.c[d];
    if (d == 4 && A.diag) v += __ldg(A.diag + i);
    return v;
}

// load a CTA-0 level operator into planar shared memory
template <int NX>
__device__ void c0_load(const Op9& A, const C0Level<NX>& L)
{
    using G = FullG<NX>;
    const long long n = (long long)NX * NX;
    for (int i = threadIdx.x; i < G::S; i += blockDim.x) L.x[i] = 0.0; // padding stays zero
    // off-diagonal planes: asynchronous global -> shared copies (all in flight;
    // completed by cp.async.wait_all before the cluster barrier that ends loading)
    for (int i = threadIdx.x; i < NX * NX; i += blockDim.x) {
        const int gy = i / NX, gx = i - gy * NX;
        const int me = G::xi(gx, gy);
#pragma unroll
        for (int d = 0; d < 9; ++d) {
            if (d == 4) continue;
            if (A.coef) {
                const unsigned dst = (unsigned)__cvta_generic_to_shared(L.coef + d * G::S + me);
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst),
                             "l"(A.coef + d * n + i)
                             : "memory");
            } else {
                L.coef[d * G::S + me] = A.c[d];
            }
        }
        const double v = op_entry(A, 4, n, i);
        L.coef[4 * G::S + me] = v;
        L.inv[me] = 1.0 / v;
    }
}

__device__ int g_probe_on = 0;
// copy of g_probe_on taken once per launch: a global load per probe would stall
// thread 0 (and through the next barrier, the CTA) even with probes disabled
__shared__ int s_probe_on;
__device__ unsigned long long g_tprobe[64];
__device__ __forceinline__ void probe(unsigned rank, int i)
{
    if (threadIdx.x == 0 && rank < 2 && s_probe_on) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g_tprobe[rank * 32 + i] = t;
    }
}

// CTA-0 V-cycle for levels of size NX, NX/2, ..., 3 (LU at 3x3)
template <int NX>
struct C0Cycle {
    static constexpr int DEPTH = 1 + C0Cycle<NX / 2>::DEPTH;
    static constexpr size_t doubles() { return 13 * (size_t)FullG<NX>::S + C0Cycle<NX / 2>::doubles(); }
    __device__ static void layout(double* base, C0Level<NX>& L)
    {
        constexpr int S = FullG<NX>::S;
        L.coef = base;
        L.x = base + 9 * S;
        L.b = L.x + S;
        L.inv = L.b + S;
        L.r = L.inv + S;
    }
    __device__ static void load(double* base, const BottomArgs& a, int k)
    {
        C0Level<NX> L;
        layout(base, L);
        c0_load<NX>(a.ops[k], L);
        C0Cycle<NX / 2>::load(base + 13 * FullG<NX>::S, a, k + 1);
    }
    __device__ __noinline__ static void run(double* base, const double* lu, const int* perm, int pre,
                                            int post)
    {
        constexpr int NC = NX / 2;
        constexpr int PB = 8 + 4 * (3 - DEPTH); // probe slots: level 31 -> 8.., 15 -> 12.., 7 -> 16..
        C0Level<NX> L;
        layout(base, L);
        double* cbase = base + 13 * FullG<NX>::S;
        C0Level<NC> Lc;
        C0Cycle<NC>::layout(cbase, Lc);
        for (int s = 0; s < pre; ++s) c0_sweep<true, NX>(L);
        probe(0, PB);
        c0_residual<NX>(L);
        for (int I = threadIdx.x; I < NC * NC; I += blockDim.x) {
            const int cy = I / NC, cx = I - cy * NC;
            const int ci = FullG<NC>::xi(cx, cy);
            Lc.b[ci] = restrict_from([&](int gx, int gy) { return L.r[FullG<NX>::xi(gx, gy)]; }, cx, cy);
            Lc.x[ci] = 0.0;
        }
        __syncthreads();
        probe(0, PB + 1);
        C0Cycle<NC>::run(cbase, lu, perm, pre, post);
        probe(0, PB + 2);
        for (int i = threadIdx.x; i < NX * NX; i += blockDim.x) {
            const int gy = i / NX, gx = i - gy * NX;
            const int me = FullG<NX>::xi(gx, gy);
            L.x[me] += prolong_from<NC>([&](int u, int v) { return Lc.x[FullG<NC>::xi(u, v)]; }, gx, gy);
        }
        __syncthreads();
        for (int s = 0; s < post; ++s) c0_sweep<false, NX>(L);
        probe(0, PB + 3);
    }
};

template <>
struct C0Cycle<3> { // level 2: dense 9x9 LU solve (DenseFactor::solve), factor in shared memory
    static constexpr int DEPTH = 0;
    static constexpr size_t doubles() { return 13 * (size_t)FullG<3>::S; }
    __device__ static void layout(double* base, C0Level<3>& L)
    {
        constexpr int S = FullG<3>::S;
        L.coef = base;
        L.x = base + 9 * S;
        L.b = L.x + S;
        L.inv = L.b + S;
        L.r = L.inv + S;
    }
    __device__ static void load(double*, const BottomArgs&, int) {}
    __device__ static void run(double* base, const double* lu, const int* perm, int, int)
    {
        C0Level<3> L;
        layout(base, L);
        if (threadIdx.x == 0) {
            double y[9];
#pragma unroll
            for (int i = 0; i < 9; ++i) {
                const int q = perm[i];
                y[i] = L.b[FullG<3>::xi(q % 3, q / 3)];
            }
#pragma unroll
            for (int i = 0; i < 9; ++i)
#pragma unroll
                for (int k2 = 0; k2 < i; ++k2) y[i] -= lu[k2 * 9 + i] * y[k2];
#pragma unroll
            for (int i = 8; i >= 0; --i) {
#pragma unroll
                for (int k2 = i + 1; k2 < 9; ++k2) y[i] -= lu[k2 * 9 + i] * y[k2];
                y[i] /= lu[i * 9 + i];
            }
#pragma unroll
            for (int i = 0; i < 9; ++i) L.x[FullG<3>::xi(i % 3, i / 3)] = y[i];
        }
        __syncthreads();
    }
};

// ----------------------------------------------------------- shared layout
template <int TOP>
struct Lay {
    using G0 = SlabG<(1 << TOP) - 1, TOP == 7 ? 8 : 4>; // top slab level
    using G1 = SlabG<63, 4>;                             // level 6 below a level-7 top
    static constexpr bool S1 = TOP == 7;
    static constexpr int BARS = 0; // 8 mbarriers (4 per slab level)
    static constexpr int X0 = BARS + 8;
    static constexpr int R0 = X0 + G0::XS;
    static constexpr int X1 = R0 + G0::RS;
    static constexpr int R1 = X1 + (S1 ? G1::XS : 0);
    static constexpr int C1 = R1 + (S1 ? G1::RS : 0); // coef [4 colours][9][GROUP1]
    static constexpr int I1 = C1 + (S1 ? 36 * G1::GROUP : 0);
    static constexpr int B1 = I1 + (S1 ? 4 * G1::GROUP : 0);
    static constexpr int RED = B1 + (S1 ? 4 * G1::GROUP : 0); // cluster reduction slots
    static constexpr int LU = RED + kCS;                      // 81 LU + 9 perm (as int)
    static constexpr int C0BASE = LU + 96;                    // CTA-0 levels (31, 15, 7, 3)
    static constexpr size_t total() { return (size_t)C0BASE + C0Cycle<31>::doubles(); }
};

template <int TOP>
__global__ void __launch_bounds__(kCT, 1)
    k_bottom_cluster(BottomArgs a, const double* __restrict__ bg, double* __restrict__ xg,
                     int cycles, int pre, int post, int check, double* state, int* flags)
{
    using Ly = Lay<TOP>;
    using G0 = typename Ly::G0;
    using G1 = typename Ly::G1;
    constexpr int NX0 = G0::NX, RP0 = G0::RP;
    constexpr int NC = 31; // first CTA-0 level
    extern __shared__ double sm[];
    __shared__ double red[33];
    cg::cluster_group cl = cg::this_cluster();
    const int w = (int)cl.block_rank();
    if (threadIdx.x == 0) s_probe_on = g_probe_on;
    __syncthreads();
    probe(w, 0);

    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + Ly::BARS);
    double* x0 = sm + Ly::X0;
    double* r0s = sm + Ly::R0;
    double* x1 = sm + Ly::X1;
    double* r1s = sm + Ly::R1;
    double* c1 = sm + Ly::C1;
    double* i1 = sm + Ly::I1;
    double* b1 = sm + Ly::B1;
    double* lus = sm + Ly::LU;
    int* perms = reinterpret_cast<int*>(lus + 81);
    double* c0base = sm + Ly::C0BASE;
    C0Level<NC> L5;
    C0Cycle<NC>::layout(c0base, L5);

    const Own<G0> o0(w);
    const Own<G1> o1(w);
    Halo<G0> H0;
    H0.setup(bars, x0, w);
    Halo<G1> H1;
    H1.setup(bars + 4, x1, w);
    if (threadIdx.x == 0) {
        H0.init_barriers();
        if constexpr (Ly::S1) H1.init_barriers();
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }

    // ---- load: the top level's four rows per thread into registers, the rest into shared memory
    double ra[4][9], rinv[4], rb[4];
    {
        const Op9& A = a.ops[0];
        const long long n = (long long)NX0 * NX0;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            if (o0.valid(c)) {
                const long long gi = (long long)o0.gy(c) * NX0 + o0.gx(c);
#pragma unroll
                for (int d = 0; d < 9; ++d) ra[c][d] = op_entry(A, d, n, gi);
                rinv[c] = 1.0 / ra[c][4];
                rb[c] = bg[gi];
            } else {
#pragma unroll
                for (int d = 0; d < 9; ++d) ra[c][d] = 0.0;
                rinv[c] = rb[c] = 0.0;
            }
        }
        for (int i = threadIdx.x; i < G0::XS; i += blockDim.x) x0[i] = 0.0;
    }
    if constexpr (Ly::S1) {
        const Op9& A = a.ops[1];
        const long long n = (long long)G1::NX * G1::NX;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            if (o1.valid(c)) {
                const long long gi = (long long)o1.gy(c) * G1::NX + o1.gx(c);
#pragma unroll
                for (int d = 0; d < 9; ++d) {
                    const double v = op_entry(A, d, n, gi);
                    c1[(c * 9 + d) * G1::GROUP + threadIdx.x] = v;
                    if (d == 4) i1[o1.slot(c)] = 1.0 / v;
                }
            }
        }
    }
    if (w == 0) {
        C0Cycle<NC>::load(c0base, a, Ly::S1 ? 2 : 1);
        if (threadIdx.x < 81) lus[threadIdx.x] = a.lu[threadIdx.x];
        if (threadIdx.x < 9) perms[threadIdx.x] = a.perm[threadIdx.x];
        asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
    }
    cl.sync();
    probe(w, 1);

    // GS update of the thread's colour-c top-level node (register rows)
    auto upd0 = [&](int c) -> double {
        double s = rb[c];
#pragma unroll
        for (int d = 0; d < 9; ++d) {
            if (d == 4) continue;
            s -= ra[c][d] * xnb(x0, o0, c, d % 3 - 1, d / 3 - 1);
        }
        return s * rinv[c];
    };
    auto upd1 = [&](int c) -> double {
        double s = b1[o1.slot(c)];
#pragma unroll
        for (int d = 0; d < 9; ++d) {
            if (d == 4) continue;
            s -= c1[(c * 9 + d) * G1::GROUP + threadIdx.x] * xnb(x1, o1, c, d % 3 - 1, d / 3 - 1);
        }
        return s * i1[o1.slot(c)];
    };
    // cluster-wide sum of per-thread values; the result is valid in CTA 0 thread 0
    auto cluster_sum = [&](double v) -> double {
        v = block_sum(v, red);
        if (threadIdx.x == 0) cl.map_shared_rank(sm + Ly::RED, 0)[w] = v;
        cl.sync();
        double tot = 0.0;
        if (w == 0 && threadIdx.x == 0)
            for (int q = 0; q < kCS; ++q) tot += sm[Ly::RED + q];
        cl.sync();
        return tot;
    };
    // residual of the top level at the thread's nodes (stored for the restriction); returns sum r^2
    auto top_residual = [&]() -> double {
        H0.ensure_all();
        double r2 = 0.0;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            if (o0.valid(c)) {
                double s = 0.0;
#pragma unroll
                for (int d = 0; d < 9; ++d) s += ra[c][d] * xnb(x0, o0, c, d % 3 - 1, d / 3 - 1);
                const double r = rb[c] - s;
                r0s[(o0.gy(c) - RP0 * w) * NX0 + o0.gx(c)] = r;
                r2 += r * r;
            }
        }
        return r2;
    };
    // prolongate a coarse correction into a slab level: own nodes, then the two
    // halo rows recomputed from the same parents (the neighbour does the same)
    auto prolong_slab = [&](auto geo, double* xs, const auto& own, const auto& cxv) {
        using GG = decltype(geo);
        constexpr int NXF = GG::NX, RPF = GG::RP, NXC = NXF / 2;
#pragma unroll
        for (int c = 0; c < 4; ++c)
            if (own.valid(c)) xs[own.me(c)] += prolong_from<NXC>(cxv, own.gx(c), own.gy(c));
        const int t = threadIdx.x;
        if (t < 2 * NXF) {
            const int gx = t % NXF, side = t / NXF;
            const int lr = side ? RPF + 1 : 0;
            const int gy = RPF * w + lr - 1;
            if (gy >= 0 && gy < NXF) xs[GG::xi(gx, lr)] += prolong_from<NXC>(cxv, gx, gy);
        }
        cl.sync(); // neighbours finish reading their old halo values before new pushes
    };

    double prev = 0.0;
    if (check) {
        double b2 = 0.0;
#pragma unroll
        for (int c = 0; c < 4; ++c) b2 += rb[c] * rb[c];
        prev = sqrt(cluster_sum(b2));
    }

    for (int cyc = 0; cyc < cycles; ++cyc) {
        // ===================== top slab level: pre-smoothing, residual
        for (int s = 0; s < pre; ++s) slab_sweep<true>(x0, H0, o0, upd0);
        top_residual();
        cl.sync();
        probe(w, 2);
        if constexpr (Ly::S1) {
            // restrict into this CTA's level-6 rows (fine row 2J+2 may be remote)
            auto fr0 = [&](int gx, int gy) -> double {
                const int owner = gy / RP0;
                const double* rr = owner == w ? r0s : cl.map_shared_rank(r0s, (unsigned)owner);
                return rr[(gy - owner * RP0) * NX0 + gx];
            };
#pragma unroll
            for (int c = 0; c < 4; ++c)
                if (o1.valid(c)) b1[o1.slot(c)] = restrict_from(fr0, o1.gx(c), o1.gy(c));
            for (int i = threadIdx.x; i < G1::XS; i += blockDim.x) x1[i] = 0.0;
            cl.sync();
            for (int s = 0; s < pre; ++s) slab_sweep<true>(x1, H1, o1, upd1);
            H1.ensure_all();
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                if (o1.valid(c)) {
                    double sum = 0.0;
#pragma unroll
                    for (int d = 0; d < 9; ++d)
                        sum += c1[(c * 9 + d) * G1::GROUP + threadIdx.x] * xnb(x1, o1, c, d % 3 - 1, d / 3 - 1);
                    r1s[(o1.gy(c) - G1::RP * w) * G1::NX + o1.gx(c)] = b1[o1.slot(c)] - sum;
                }
            }
            cl.sync();
            probe(w, 3);
        }
        // restrict the last slab level into CTA 0's level-5 b (distributed, DSM stores)
        {
            using GS = std::conditional_t<Ly::S1, G1, G0>;
            const double* rl = Ly::S1 ? r1s : r0s;
            auto frs = [&](int gx, int gy) -> double {
                const int owner = gy / GS::RP;
                const double* rr = owner == w ? rl : cl.map_shared_rank(rl, (unsigned)owner);
                return rr[(gy - owner * GS::RP) * GS::NX + gx];
            };
            double* b5 = cl.map_shared_rank(L5.b, 0);
            double* x5 = cl.map_shared_rank(L5.x, 0);
            // coarse rows J whose centre fine row 2J+1 lies in this CTA's band
            const int J0 = (GS::RP * w) / 2, J1 = min((GS::RP * w + GS::RP) / 2, NC);
            for (int i = threadIdx.x; i < (J1 - J0) * NC; i += blockDim.x) {
                const int J = J0 + i / NC, I = i - (i / NC) * NC;
                const int ci = FullG<NC>::xi(I, J);
                b5[ci] = restrict_from(frs, I, J);
                x5[ci] = 0.0;
            }
        }
        cl.sync();
        probe(w, 4);
        // ===================== CTA-0 levels and the LU solve
        if (w == 0) C0Cycle<NC>::run(c0base, lus, perms, pre, post);
        cl.sync();
        probe(w, 5);
        // ===================== prolongations and post-smoothing
        {
            const double* c5x = cl.map_shared_rank(L5.x, 0);
            auto cx5 = [&](int u, int v) { return c5x[FullG<NC>::xi(u, v)]; };
            if constexpr (Ly::S1) {
                prolong_slab(G1{}, x1, o1, cx5);
                for (int s = 0; s < post; ++s) slab_sweep<false>(x1, H1, o1, upd1);
                H1.ensure_all();
                // level-7 parents lie in this CTA's level-6 band or its halo rows
                auto cx6 = [&](int u, int v) { return x1[G1::xi(u, v - G1::RP * w + 1)]; };
                prolong_slab(G0{}, x0, o0, cx6);
            } else {
                prolong_slab(G0{}, x0, o0, cx5);
            }
        }
        probe(w, 6);
        for (int s = 0; s < post; ++s) slab_sweep<false>(x0, H0, o0, upd0);
        probe(w, 7);
        if (check) {
            const double res = sqrt(cluster_sum(top_residual()));
            if (w == 0 && threadIdx.x == 0 && res > 10.0 * prev) atomicOr(flags, kErrMgDiverged);
            prev = res;
        }
        H0.ensure_all();
    }
#pragma unroll
    for (int c = 0; c < 4; ++c)
        if (o0.valid(c)) xg[(long long)o0.gy(c) * NX0 + o0.gx(c)] = x0[o0.me(c)];
    if (check && state && w == 0 && threadIdx.x == 0) state[0] = prev;
    cl.sync(); // no CTA exits while a neighbour may still address its shared memory
}

template <int TOP>
cudaLaunchConfig_t cluster_cfg(cudaStream_t s, cudaLaunchAttribute* at)
{
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(kCS);
    cfg.blockDim = dim3(kCT);
    cfg.dynamicSmemBytes = Lay<TOP>::total() * sizeof(double);
    cfg.stream = s;
    at->id = cudaLaunchAttributeClusterDimension;
    at->val.clusterDim.x = kCS;
    at->val.clusterDim.y = 1;
    at->val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cfg;
}

template <int TOP>
bool set_attrs()
{
    return cudaFuncSetAttribute(k_bottom_cluster<TOP>,
                                cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess &&
           cudaFuncSetAttribute(k_bottom_cluster<TOP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)(Lay<TOP>::total() * sizeof(double))) == cudaSuccess;
}

template <int TOP>
void launch_top(cudaStream_t s, const BottomArgs& a, const double* b, double* x, int cycles,
                int pre, int post, bool check, double* state, int* flags)
{
    static const bool attr = set_attrs<TOP>();
    (void)attr;
    cudaLaunchAttribute at{};
    cudaLaunchConfig_t cfg = cluster_cfg<TOP>(s, &at);
    note_launch();
    cudaLaunchKernelEx(&cfg, k_bottom_cluster<TOP>, a, b, x, cycles, pre, post, check ? 1 : 0,
                       state, flags);
}

static_assert(Lay<7>::total() * sizeof(double) <= 220 * 1024, "cluster layout exceeds shared memory");

} // namespace

void cluster_probes(int enable, unsigned long long* out64)
{
    cudaMemcpyToSymbol(g_probe_on, &enable, sizeof(int));
    if (out64) cudaMemcpyFromSymbol(out64, g_tprobe, 64 * sizeof(unsigned long long));
}

bool cluster_bottom_supported()
{
    static const bool supported = [] {
        bool ok = set_attrs<7>() && set_attrs<6>();
        if (ok) {
            cudaLaunchAttribute at{};
            cudaLaunchConfig_t cfg = cluster_cfg<7>(nullptr, &at);
            int nclusters = 0;
            ok = cudaOccupancyMaxActiveClusters(&nclusters, k_bottom_cluster<7>, &cfg) == cudaSuccess &&
                 nclusters > 0;
        }
        cudaGetLastError();
        return ok;
    }();
    return supported;
}

void launch_bottom_cluster(cudaStream_t s, const ClusterArgs& a, const double* b, double* x,
                           int cycles, int pre, int post, bool check, double* state, int* flags)
{
    if (a.ops[0].nx == 127) launch_top<7>(s, a, b, x, cycles, pre, post, check, state, flags);
    else if (a.ops[0].nx == 63) launch_top<6>(s, a, b, x, cycles, pre, post, check, state, flags);
    else throw std::runtime_error("cluster bottom: top level must be 6 or 7");
}

} // namespace ocb
