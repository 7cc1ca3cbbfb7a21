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
constexpr int kCopN = 225;   // level-4 nodes (15 x 15): dense V-cycle operator below level 5
constexpr int kCopRows = 15; // rows of it per CTA 1..15

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
template <int NX_, int RP_, int NPT_ = 1>
struct SlabG {
    static constexpr int NX = NX_, RP = RP_, NPT = NPT_; // NPT node positions per colour per thread
    static constexpr int WX = (NX + 1) / 2;     // columns per colour row
    static constexpr int SX = WX + 1;           // padded row stride
    static constexpr int RH = RP / 2;           // colour rows per band
    static constexpr int PS = (RH + 1) * SX;    // plane size (incl. the halo rows)
    static constexpr int XS = 4 * PS;           // planar x with halos
    static constexpr int GROUP = RH * WX;       // threads owning nodes (one per colour)
    static constexpr int RS = RP * NX;          // row-major residual of own rows
    static_assert(RP % 2 == 0, "even row bands keep the colour parity per CTA");
    static_assert(GROUP <= NPT * kCT, "NPT nodes per colour per thread");
    static_assert(NPT == 1 || GROUP == NPT * kCT, "multi-position levels fill every thread");
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

// The NPT nodes per colour of a thread on a multi-position slab level (the
// level-8 top): thread t owns column t mod WX of the NPT consecutive colour
// rows NPT (t / WX) + m, so a warp covers 32 consecutive columns of one colour
// row and a thread's positions m, m+1 share their in-between grid row (three
// of the eight neighbour loads).
template <class G>
struct OwnM {
    static constexpr int N = G::NPT;
    int cc[N], rr[N], q[N];
    int r0;
    __device__ explicit OwnM(int w)
    {
#pragma unroll
        for (int m = 0; m < N; ++m) {
            rr[m] = N * (threadIdx.x / G::WX) + m;
            cc[m] = threadIdx.x % G::WX;
            q[m] = rr[m] * G::SX + cc[m];
        }
        r0 = G::RP * w;
    }
    __device__ __forceinline__ int gx(int m, int c) const { return 2 * cc[m] + (c & 1); }
    __device__ __forceinline__ int gy(int m, int c) const { return r0 + 2 * rr[m] + (c >> 1); }
    __device__ __forceinline__ bool valid(int m, int c) const { return gx(m, c) < G::NX && gy(m, c) < G::NX; }
    __device__ __forceinline__ int me(int m, int c) const { return q[m] + G::nb(c, 0, 0); }
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
    // consume the pending colour-c exchange: every thread keeps the phase
    // bookkeeping, only `waiter` threads (those reading that halo row) spin on
    // the mbarrier, and one of them (`armer`) re-arms the next phase
    __device__ __forceinline__ void ensure(int c, bool waiter = true, bool armer = threadIdx.x == 0)
    {
        if (!((pend >> c) & 1u)) return;
        pend &= ~(1u << c);
        if (!(c < 2 ? has_dn() : has_up())) return;
        if (waiter) mbar_wait(bar + 8 * c, (par >> c) & 1u);
        par ^= 1u << c;
        if (armer) mbar_expect(bar + 8 * c, G::seg_bytes(c));
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
    // multi-position levels: the node at column gx of colour row rr
    __device__ __forceinline__ void push_at(int gx, int rr, double v, int c) const
    {
        if (c < 2 && rr == 0 && has_up())
            st_async(mapa(xs + 8u * G::xi(gx, G::RP + 1), (uint32_t)(w - 1)), v,
                     mapa(bar + 8 * c, (uint32_t)(w - 1)));
        if (c >= 2 && rr == G::RH - 1 && has_dn())
            st_async(mapa(xs + 8u * G::xi(gx, 0), (uint32_t)(w + 1)), v,
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
        // first-row nodes read the upper halo (colours 2, 3), last-row nodes the
        // lower one (colours 0, 1); the other rows update without waiting
        const bool edge = c < 2 ? o.rr == 0 : o.rr == G::RH - 1;
        const bool armer = edge && o.cc == 0;
        // every owning thread updates (warp-uniform): a position outside the
        // domain has zero b, coefficients and 1/a_ii, so it rewrites its zero pad
        double v = 0.0;
        if (o.thr && !edge) {
            v = upd(c);
            xs[o.me(c)] = v;
        }
        H.ensure(c < 2 ? 2 : 0, edge, armer);
        H.ensure(c < 2 ? 3 : 1, edge, armer);
        if (o.thr && edge) {
            v = upd(c);
            xs[o.me(c)] = v;
        }
        __syncthreads(); // CTA-local visibility; every halo read of this pass is done
        if (o.valid(c)) H.push(o, v, c);
        H.passed(c);
    }
}

// The same on a multi-position level: upd(m, c) for the thread's nodes m.
template <bool FWD, class G, typename U>
__device__ __forceinline__ void slab_sweep_m(double* xs, Halo<G>& H, const OwnM<G>& o, const U& upd)
{
#pragma unroll
    for (int p = 0; p < 4; ++p) {
        const int c = FWD ? p : 3 - p;
        // (waiting only in the edge warps and updating the other positions first,
        // as slab_sweep does, costs registers here and measured slower)
        H.ensure(c < 2 ? 2 : 0);
        H.ensure(c < 2 ? 3 : 1);
        double v[G::NPT]; // positions outside the domain compute 0 (zero b and 1/a_ii)
#pragma unroll
        for (int m = 0; m < G::NPT; ++m) v[m] = upd(m, c);
#pragma unroll
        for (int m = 0; m < G::NPT; ++m) xs[o.me(m, c)] = v[m];
        __syncthreads();
#pragma unroll
        for (int m = 0; m < G::NPT; ++m)
            if (o.valid(m, c)) H.push_at(o.gx(m, c), o.rr[m], v[m], c);
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
__device__ void c0_load(const Op9& A, const C0Level<NX>& L, long long shift = 0)
{
    using G = FullG<NX>;
    const long long n = (long long)NX * NX;
    const double* coef = A.coef ? A.coef + shift : nullptr; // batch element of a chained launch
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
                             "l"(coef + d * n + i)
                             : "memory");
            } else {
                L.coef[d * G::S + me] = A.c[d];
            }
        }
        const double v = op_entry(A, 4, n, i + shift);
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
    // x and b first: below the top CTA-0 level the cluster kernel keeps only them
    __device__ static void layout(double* base, C0Level<NX>& L)
    {
        constexpr int S = FullG<NX>::S;
        L.x = base;
        L.b = base + S;
        L.inv = base + 2 * S;
        L.r = base + 3 * S;
        L.coef = base + 4 * S;
    }
    __device__ static void load(double* base, const BottomArgs& a, int k)
    {
        C0Level<NX> L;
        layout(base, L);
        c0_load<NX>(a.ops[k], L);
        C0Cycle<NX / 2>::load(base + 13 * FullG<NX>::S, a, k + 1);
    }
    __device__ static void load_top(double* base, const BottomArgs& a, int k, long long shift = 0) // this level only
    {
        C0Level<NX> L;
        layout(base, L);
        c0_load<NX>(a.ops[k], L, shift);
    }
    // pre-smoothing, residual and restriction into the next level's b (x zeroed)
    __device__ static void run_pre(double* base, int pre)
    {
        constexpr int NC = NX / 2;
        constexpr int PB = 8 + 4 * (3 - DEPTH); // probe slots: level 31 -> 8.., 15 -> 12.., 7 -> 16..
        C0Level<NX> L;
        layout(base, L);
        C0Level<NC> Lc;
        C0Cycle<NC>::layout(base + 13 * FullG<NX>::S, Lc);
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
    }
    // prolongation of the next level's x and post-smoothing
    __device__ static void run_post(double* base, int post)
    {
        constexpr int NC = NX / 2;
        constexpr int PB = 8 + 4 * (3 - DEPTH);
        C0Level<NX> L;
        layout(base, L);
        C0Level<NC> Lc;
        C0Cycle<NC>::layout(base + 13 * FullG<NX>::S, Lc);
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
    __device__ __noinline__ static void run(double* base, const double* lu, const int* perm, int pre,
                                            int post)
    {
        run_pre(base, pre);
        C0Cycle<NX / 2>::run(base + 13 * FullG<NX>::S, lu, perm, pre, post);
        run_post(base, post);
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
// TOP = 8: a constant-stencil (+ diagonal) level 8 in 16-row bands (4 nodes
// per colour per thread; x in shared memory, b and 1/a_ii in registers) above
// the level-7 structure. Level-8 residual rows share space with the level-7
// and level-6 residuals (never live at the same time).
template <int TOP>
struct Lay {
    static constexpr bool S8 = TOP == 8;
    static constexpr bool S1 = TOP >= 7;
    using G8 = SlabG<255, 16, 4>;                        // level 8 (TOP = 8)
    using G0 = SlabG<S1 ? 127 : 63, S1 ? 8 : 4>;         // level 7 (TOP 7, 8) or 6 (TOP 6)
    using G1 = SlabG<63, 4>;                             // level 6 below a level-7 slab
    static constexpr int BARS = 0;                       // 12 mbarriers (4 per slab level)
    static constexpr int X8 = BARS + 12;
    static constexpr int X0 = X8 + (S8 ? G8::XS : 0);
    static constexpr int RT = X0 + G0::XS;               // residual rows
    static constexpr int R0 = RT;
    static constexpr int R1 = R0 + G0::RS;
    static constexpr int RTS = (S8 && G8::RS > G0::RS + G1::RS) ? G8::RS : G0::RS + (S1 ? G1::RS : 0);
    static constexpr int X1 = RT + RTS;
    static constexpr int C1 = X1 + (S1 ? G1::XS : 0); // coef [4 colours][9][GROUP1]
    static constexpr int I1 = C1 + (S1 ? 36 * G1::GROUP : 0);
    static constexpr int B1 = I1 + (S1 ? 4 * G1::GROUP : 0);
    static constexpr int RED = B1 + (S1 ? 4 * G1::GROUP : 0); // cluster reduction slots
    static constexpr int C0BASE = RED + kCS;                  // CTA 0: level 5 + level-4 x, b
    static constexpr size_t total() { return (size_t)C0BASE + 13 * FullG<31>::S + 2 * FullG<15>::S; }
};

template <int TOP>
__global__ void __launch_bounds__(kCT, 1)
    k_bottom_cluster(BottomArgs a, const double* __restrict__ bg0, double* __restrict__ xg0,
                     int cycles, int pre, int post, int check, double* state, int* flags, ChainArgs ch)
{
    using Ly = Lay<TOP>;
    using G8 = typename Ly::G8;
    using G0 = typename Ly::G0;
    using G1 = typename Ly::G1;
    constexpr bool S8 = Ly::S8;
    constexpr int NX0 = G0::NX, RP0 = G0::RP;
    constexpr int NC = 31; // first CTA-0 level
    constexpr int K0 = S8 ? 1 : 0; // ops index of the G0 level
    extern __shared__ double sm[];
    __shared__ double red[33];
    cg::cluster_group cl = cg::this_cluster();
    const int w = (int)cl.block_rank();
    if (threadIdx.x == 0) s_probe_on = g_probe_on;
    __syncthreads();
    probe(w, 0);

    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + Ly::BARS);
    double* x8 = sm + Ly::X8;
    double* r8s = sm + Ly::RT;
    double* x0 = sm + Ly::X0;
    double* r0s = sm + Ly::R0;
    double* x1 = sm + Ly::X1;
    double* r1s = sm + Ly::R1;
    double* c1 = sm + Ly::C1;
    double* i1 = sm + Ly::I1;
    double* b1 = sm + Ly::B1;
    double* c0base = sm + Ly::C0BASE;
    C0Level<NC> L5;
    C0Cycle<NC>::layout(c0base, L5);

    const OwnM<G8> o8(w);
    const Own<G0> o0(w);
    const Own<G1> o1(w);
    Halo<G0> H0;
    H0.setup(bars, x0, w);
    Halo<G1> H1;
    H1.setup(bars + 4, x1, w);
    Halo<G8> H8;
    H8.setup(bars + 8, x8, w);
    if (threadIdx.x == 0) {
        H0.init_barriers();
        if constexpr (Ly::S1) H1.init_barriers();
        if constexpr (S8) H8.init_barriers();
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }

    // A chained launch (heat time blocks, TimeSchurApprox::apply_inverse,
    // timedep.cpp:268-311) solves ch.nblk batch elements one after the other:
    // element ob = blk * ch.dbt away from the first, with the right-hand side
    // b = r + M x_prev formed from the previous element's solution while it is
    // still in shared memory (own rows and up-to-date halo rows).
    const int nblk = S8 ? max(ch.nblk, 1) : 1;
#pragma unroll 1
    for (int blk = 0; blk < nblk; ++blk) {
    const long long ob = S8 ? (long long)blk * ch.dbt : 0; // batch element offset
    const double* __restrict__ bg = bg0 + ob * ch.ns;
    double* __restrict__ xg = xg0 + ob * ch.ns;
    const double* diag8 = (S8 && a.ops[0].diag) ? a.ops[0].diag + ob * ch.ns : nullptr;
    // ---- load. First the asynchronous copies (they complete while the register
    // rows below are loaded): levels <= 4 are CTAs 1..15 holding 15 rows each of
    // the dense level-4 V-cycle operator (k_coarse_op) where CTA 0 keeps level 5
    // (the region's last readers finished before the previous element's closing
    // cluster barrier)
    double* cops = c0base;
    if (w > 0) {
        const double* src = a.cop + ob * kCopN * kCopN + (size_t)kCopRows * kCopN * (w - 1);
        for (int i = threadIdx.x; i < kCopRows * kCopN; i += blockDim.x) {
            const unsigned dst = (unsigned)__cvta_generic_to_shared(cops + i);
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst), "l"(src + i) : "memory");
        }
    } else {
        C0Cycle<NC>::load_top(c0base, a, K0 + (Ly::S1 ? 2 : 1), ob * 9 * NC * NC);
    }
    // Level 8: b and 1/a_ii of the thread's 16 nodes in registers.
    double rb8[S8 ? G8::NPT : 1][4] = {}, ri8[S8 ? G8::NPT : 1][4] = {};
    if constexpr (S8) {
        const Op9& A = a.ops[0];
#pragma unroll
        for (int m = 0; m < G8::NPT; ++m)
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                rb8[m][c] = ri8[m][c] = 0.0;
                if (o8.valid(m, c)) {
                    const long long gi = (long long)o8.gy(m, c) * G8::NX + o8.gx(m, c);
                    double bv = bg[gi];
                    if (blk > 0) { // + M x_prev in op_apply_at's order (k_rhs_plus_mass)
                        double sm9 = 0.0;
#pragma unroll
                        for (int d = 0; d < 9; ++d)
                            sm9 += ch.mc[d] * x8[o8.q[m] + G8::nb(c, d % 3 - 1, d / 3 - 1)];
                        bv = bv + sm9;
                    }
                    rb8[m][c] = bv;
                    ri8[m][c] = 1.0 / (A.c[4] + (diag8 ? diag8[gi] : 0.0)); // = k_inv_diag
                }
            }
        if (blk > 0) __syncthreads(); // every read of the previous solution is done
        for (int i = threadIdx.x; i < G8::XS; i += blockDim.x) x8[i] = 0.0;
    }
    // the G0 level's four nodes per thread: coefficients, 1/a_ii, b in registers
    double ra[4][9], rinv[4], rb[4];
    {
        const Op9& A = a.ops[K0];
        const long long n = (long long)NX0 * NX0;
        const long long sh = ob * 9 * n;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            if (o0.valid(c)) {
                const long long gi = (long long)o0.gy(c) * NX0 + o0.gx(c);
#pragma unroll
                for (int d = 0; d < 9; ++d) ra[c][d] = op_entry(A, d, n, gi + sh);
                rinv[c] = 1.0 / ra[c][4];
                rb[c] = S8 ? 0.0 : bg[gi];
            } else {
#pragma unroll
                for (int d = 0; d < 9; ++d) ra[c][d] = 0.0;
                rinv[c] = rb[c] = 0.0;
            }
        }
        for (int i = threadIdx.x; i < G0::XS; i += blockDim.x) x0[i] = 0.0;
    }
    if constexpr (Ly::S1) {
        const Op9& A = a.ops[K0 + 1];
        const long long n = (long long)G1::NX * G1::NX;
        const long long sh = ob * 9 * n;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            if (o1.valid(c)) {
                const long long gi = (long long)o1.gy(c) * G1::NX + o1.gx(c);
#pragma unroll
                for (int d = 0; d < 9; ++d) {
                    const double v = op_entry(A, d, n, gi + sh);
                    c1[(c * 9 + d) * G1::GROUP + threadIdx.x] = v;
                    if (d == 4) i1[o1.slot(c)] = 1.0 / v;
                }
            } else if (o1.thr) { // outside the domain: zero row (branch-free sweeps)
#pragma unroll
                for (int d = 0; d < 9; ++d) c1[(c * 9 + d) * G1::GROUP + threadIdx.x] = 0.0;
                i1[o1.slot(c)] = 0.0;
                b1[o1.slot(c)] = 0.0;
            }
        }
    }
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory"); // level 5 / dense rows
    cl.sync();
    probe(w, 1);

    // GS update of the thread's colour-c G0 node (register rows)
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
    // level 8: constant stencil, the reference row order (k_sweep)
    auto upd8 = [&](int m, int c) -> double {
        const Op9& A = a.ops[0];
        double s = rb8[m][c];
#pragma unroll
        for (int d = 0; d < 9; ++d) {
            if (d == 4) continue;
            s -= A.c[d] * x8[o8.q[m] + G8::nb(c, d % 3 - 1, d / 3 - 1)];
        }
        return s * ri8[m][c];
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
    // residual of the G0 level at the thread's nodes (stored for the restriction); returns sum r^2
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
    // level-8 residual (k_resid_restrict's row order), stored row-major; returns sum r^2
    auto residual8 = [&]() -> double {
        H8.ensure_all();
        const Op9& A = a.ops[0];
        double r2 = 0.0;
#pragma unroll
        for (int m = 0; m < G8::NPT; ++m)
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                if (!o8.valid(m, c)) continue;
                const long long gi = (long long)o8.gy(m, c) * G8::NX + o8.gx(m, c);
                double s = 0.0;
#pragma unroll
                for (int d = 0; d < 9; ++d) {
                    double av = A.c[d];
                    if (d == 4 && diag8) av += diag8[gi];
                    s += av * x8[o8.q[m] + G8::nb(c, d % 3 - 1, d / 3 - 1)];
                }
                const double r = rb8[m][c] - s;
                r8s[(o8.gy(m, c) - G8::RP * w) * G8::NX + o8.gx(m, c)] = r;
                r2 += r * r;
            }
        return r2;
    };
    // prolongate a coarse correction into a slab level: own nodes, then the two
    // halo rows recomputed from the same parents (the neighbour does the same)
    auto prolong_halo = [&](auto geo, double* xs, const auto& cxv) {
        using GG = decltype(geo);
        constexpr int NXF = GG::NX, RPF = GG::RP, NXC = NXF / 2;
        for (int t = threadIdx.x; t < 2 * NXF; t += blockDim.x) {
            const int gx = t % NXF, side = t / NXF;
            const int lr = side ? RPF + 1 : 0;
            const int gy = RPF * w + lr - 1;
            if (gy >= 0 && gy < NXF) xs[GG::xi(gx, lr)] += prolong_from<NXC>(cxv, gx, gy);
        }
        cl.sync(); // neighbours finish reading their old halo values before new pushes
    };
    auto prolong_slab = [&](auto geo, double* xs, const auto& own, const auto& cxv) {
        using GG = decltype(geo);
        constexpr int NXC = GG::NX / 2;
#pragma unroll
        for (int c = 0; c < 4; ++c)
            if (own.valid(c)) xs[own.me(c)] += prolong_from<NXC>(cxv, own.gx(c), own.gy(c));
        prolong_halo(geo, xs, cxv);
    };

    // ===================== one V-cycle from the G0 level down (x0 holds its iterate)
    auto cycle0 = [&]() {
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
        // ===================== level 5 in CTA 0; levels <= 4 as x4 = B4 b4
        if (w == 0) C0Cycle<NC>::run_pre(c0base, pre);
        cl.sync();
        if (w > 0) { // 15 rows per CTA, 16 lanes per row, DSM in and out
            C0Level<NC / 2> L4;
            C0Cycle<NC / 2>::layout(c0base + 13 * FullG<NC>::S, L4);
            const double* b4 = cl.map_shared_rank(L4.b, 0);
            double* x4 = cl.map_shared_rank(L4.x, 0);
            double* b4l = cops + kCopRows * kCopN; // local copy of b4
            for (int j = threadIdx.x; j < kCopN; j += blockDim.x) b4l[j] = b4[FullG<NC / 2>::xi(j % 15, j / 15)];
            __syncthreads();
            const int r = threadIdx.x >> 4, ch = threadIdx.x & 15;
            double sum = 0.0;
            if (r < kCopRows) {
                const double* row = cops + r * kCopN;
#pragma unroll 2
                for (int j = ch; j < kCopN; j += 16) sum += row[j] * b4l[j];
            }
#pragma unroll
            for (int o = 8; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
            if (r < kCopRows && ch == 0) {
                const int i = kCopRows * (w - 1) + r;
                x4[FullG<NC / 2>::xi(i % 15, i / 15)] = sum;
            }
        }
        cl.sync();
        if (w == 0) C0Cycle<NC>::run_post(c0base, post);
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
                // G0 parents lie in this CTA's level-6 band or its halo rows
                auto cx6 = [&](int u, int v) { return x1[G1::xi(u, v - G1::RP * w + 1)]; };
                prolong_slab(G0{}, x0, o0, cx6);
            } else {
                prolong_slab(G0{}, x0, o0, cx5);
            }
        }
        probe(w, 6);
        for (int s = 0; s < post; ++s) slab_sweep<false>(x0, H0, o0, upd0);
        probe(w, 7);
    };

    double prev = 0.0;
    if (check) {
        double b2 = 0.0;
        if constexpr (S8) {
#pragma unroll
            for (int m = 0; m < G8::NPT; ++m)
#pragma unroll
                for (int c = 0; c < 4; ++c) b2 += rb8[m][c] * rb8[m][c];
        } else {
#pragma unroll
            for (int c = 0; c < 4; ++c) b2 += rb[c] * rb[c];
        }
        prev = sqrt(cluster_sum(b2));
    }

    for (int cyc = 0; cyc < cycles; ++cyc) {
        if constexpr (S8) {
            // ===================== level 8: pre-smoothing, residual, restriction into level 7
            probe(w, 20);
            for (int s = 0; s < pre; ++s) slab_sweep_m<true>(x8, H8, o8, upd8);
            probe(w, 21);
            residual8();
            cl.sync();
            probe(w, 22);
            {
                auto fr8 = [&](int gx, int gy) -> double {
                    const int owner = gy / G8::RP;
                    const double* rr = owner == w ? r8s : cl.map_shared_rank(r8s, (unsigned)owner);
                    return rr[(gy - owner * G8::RP) * G8::NX + gx];
                };
#pragma unroll
                for (int c = 0; c < 4; ++c)
                    rb[c] = o0.valid(c) ? restrict_from(fr8, o0.gx(c), o0.gy(c)) : 0.0;
                for (int i = threadIdx.x; i < G0::XS; i += blockDim.x) x0[i] = 0.0;
            }
            cl.sync(); // level-8 residual rows are free again (level-7 residual reuses them)
            probe(w, 23);
            cycle0();
            H0.ensure_all();
            probe(w, 24);
            // ===================== prolongation into level 8 (own nodes + halo rows), post-smoothing
            auto cx7 = [&](int u, int v) { return x0[G0::xi(u, v - G0::RP * w + 1)]; };
#pragma unroll
            for (int m = 0; m < G8::NPT; ++m)
#pragma unroll
                for (int c = 0; c < 4; ++c)
                    if (o8.valid(m, c)) x8[o8.me(m, c)] += prolong_from<127>(cx7, o8.gx(m, c), o8.gy(m, c));
            prolong_halo(G8{}, x8, cx7);
            probe(w, 25);
            for (int s = 0; s < post; ++s) slab_sweep_m<false>(x8, H8, o8, upd8);
            probe(w, 26);
            if (check) {
                const double res = sqrt(cluster_sum(residual8()));
                if (w == 0 && threadIdx.x == 0 && res > 10.0 * prev) atomicOr(flags, kErrMgDiverged);
                prev = res;
            }
            H8.ensure_all();
        } else {
            cycle0();
            if (check) {
                const double res = sqrt(cluster_sum(top_residual()));
                if (w == 0 && threadIdx.x == 0 && res > 10.0 * prev) atomicOr(flags, kErrMgDiverged);
                prev = res;
            }
            H0.ensure_all();
        }
    }
    if constexpr (S8) {
#pragma unroll
        for (int m = 0; m < G8::NPT; ++m)
#pragma unroll
            for (int c = 0; c < 4; ++c)
                if (o8.valid(m, c)) xg[(long long)o8.gy(m, c) * G8::NX + o8.gx(m, c)] = x8[o8.me(m, c)];
    } else {
#pragma unroll
        for (int c = 0; c < 4; ++c)
            if (o0.valid(c)) xg[(long long)o0.gy(c) * NX0 + o0.gx(c)] = x0[o0.me(c)];
    }
    if (check && state && w == 0 && threadIdx.x == 0) state[0] = prev;
    cl.sync(); // no CTA exits (or reloads) while a neighbour may still address its shared memory
    } // chained batch elements
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
                int pre, int post, bool check, double* state, int* flags, const ChainArgs& ch)
{
    static const bool attr = set_attrs<TOP>();
    (void)attr;
    cudaLaunchAttribute at{};
    cudaLaunchConfig_t cfg = cluster_cfg<TOP>(s, &at);
    note_launch();
    cudaLaunchKernelEx(&cfg, k_bottom_cluster<TOP>, a, b, x, cycles, pre, post, check ? 1 : 0,
                       state, flags, ch);
}

static_assert(Lay<7>::total() * sizeof(double) <= 220 * 1024, "cluster layout exceeds shared memory");
static_assert(Lay<8>::total() * sizeof(double) + 33 * 8 + 4 <= 227 * 1024, "level-8 layout exceeds shared memory");
static_assert((size_t)kCopRows * kCopN + kCopN <= C0Cycle<31>::doubles(), "dense operator slice exceeds the CTA-0 region");

// Dense operator of the levels <= 4 of a V-cycle (zero initial guess, `pre` /
// `post` 4-colour sweeps, LU at level 2): column j = the cycle applied to e_j,
// by the same CTA-0 code the cluster kernel ran there. out[bt][i * 225 + j].
// The cycle is linear in its right-hand side, so B4 b equals the cycle's
// result up to the order of the final sums.
__global__ void __launch_bounds__(64) k_coarse_op(BottomArgs a, int pre, int post, double* out)
{
    extern __shared__ double sm[];
    constexpr int NX = 15;
    using G = FullG<NX>;
    const int j = blockIdx.x, bt = blockIdx.y, t = threadIdx.x;
    if (t == 0) s_probe_on = 0;
#pragma unroll
    for (int k = 0; k < 2; ++k) a.ops[k].coef += (size_t)bt * 9 * a.ops[k].nx * a.ops[k].nx;
    double* lus = sm + C0Cycle<NX>::doubles();
    int* perms = reinterpret_cast<int*>(lus + 81);
    C0Cycle<NX>::load(sm, a, 0);
    for (int i = t; i < 81; i += blockDim.x) lus[i] = a.lu[81 * (size_t)bt + i];
    if (t < 9) perms[t] = a.perm[9 * (size_t)bt + t];
    C0Level<NX> L;
    C0Cycle<NX>::layout(sm, L);
    for (int i = t; i < G::S; i += blockDim.x) L.b[i] = 0.0;
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
    __syncthreads();
    if (t == 0) L.b[G::xi(j % NX, j / NX)] = 1.0;
    __syncthreads();
    C0Cycle<NX>::run(sm, lus, perms, pre, post);
    for (int i = t; i < kCopN; i += blockDim.x)
        out[(size_t)bt * kCopN * kCopN + (size_t)i * kCopN + j] = L.x[G::xi(i % NX, i / NX)];
}

} // namespace

void cluster_probes(int enable, unsigned long long* out64)
{
    cudaMemcpyToSymbol(g_probe_on, &enable, sizeof(int));
    if (out64) cudaMemcpyFromSymbol(out64, g_tprobe, 64 * sizeof(unsigned long long));
}

template <int TOP>
bool cluster_launchable()
{
    bool ok = set_attrs<TOP>();
    if (ok) {
        cudaLaunchAttribute at{};
        cudaLaunchConfig_t cfg = cluster_cfg<TOP>(nullptr, &at);
        int nclusters = 0;
        ok = cudaOccupancyMaxActiveClusters(&nclusters, k_bottom_cluster<TOP>, &cfg) == cudaSuccess &&
             nclusters > 0;
    }
    cudaGetLastError();
    return ok;
}

bool cluster_bottom_supported()
{
    static const bool supported = cluster_launchable<7>() && cluster_launchable<6>();
    return supported;
}

bool cluster_top8_supported()
{
    static const bool supported = cluster_bottom_supported() && cluster_launchable<8>();
    return supported;
}

void launch_coarse_op(cudaStream_t s, const BottomArgs& a, int batch, int pre, int post, double* out)
{
    if (a.ops[0].nx != 15 || a.ops[1].nx != 7 || !a.ops[0].coef || !a.ops[1].coef)
        throw std::runtime_error("coarse operator: levels 4 and 3 (variable stencils) expected");
    const size_t smem = (C0Cycle<15>::doubles() + 96) * sizeof(double);
    static const bool attr = cudaFuncSetAttribute(k_coarse_op, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                  (int)smem) == cudaSuccess;
    (void)attr;
    note_launch();
    k_coarse_op<<<dim3(kCopN, batch), 64, smem, s>>>(a, pre, post, out);
}

void launch_bottom_cluster(cudaStream_t s, const ClusterArgs& a, const double* b, double* x,
                           int cycles, int pre, int post, bool check, double* state, int* flags)
{
    ChainArgs one{};
    one.nblk = 1;
    if (a.ops[0].nx == 255 && !a.ops[0].coef)
        launch_top<8>(s, a, b, x, cycles, pre, post, check, state, flags, one);
    else if (a.ops[0].nx == 127) launch_top<7>(s, a, b, x, cycles, pre, post, check, state, flags, one);
    else if (a.ops[0].nx == 63) launch_top<6>(s, a, b, x, cycles, pre, post, check, state, flags, one);
    else throw std::runtime_error("cluster bottom: top level must be 6, 7 or a constant-stencil 8");
}

void launch_cluster_chain(cudaStream_t s, const ClusterArgs& a, const double* r, double* x,
                          const ChainArgs& ch, int cycles, int pre, int post, bool check,
                          double* state, int* flags)
{
    if (!(a.ops[0].nx == 255 && !a.ops[0].coef))
        throw std::runtime_error("cluster chain: a constant-stencil level-8 hierarchy expected");
    launch_top<8>(s, a, r, x, cycles, pre, post, check, state, flags, ch);
}

} // namespace ocb
