// Multi-CTA multigrid kernels for the large levels (>= 8) (sm_100a, FP64).
//
// k_sweep<TX,TY,NS,VAR>: NS symmetric-colour Gauss-Seidel sweeps (4 colour
// passes each, multigrid.cpp:44-66 restated as the 4-colour variant) over one
// TX x TY output tile per CTA. The tile plus a halo of 4*NS nodes is staged in
// shared memory with asynchronous copies (cp.async, all in flight at once) in
// a colour-planar layout (one plane per colour, so a colour pass reads every
// operand at unit stride: no bank conflicts): x, b, the reciprocal diagonal
// and, for small variable tiles, the 8 off-diagonal coefficient planes. Pass q
// then updates the colour nodes of the tile grown by 4*NS-1-q entirely from
// shared memory, so after all passes the tile is exact without inter-CTA
// synchronisation (redundant halo work). Large variable levels read their
// coefficients in the passes from a colour-split copy of per-node records
// (8 off-diagonals = four 16-byte loads from one address, then 1/a_ii;
// Op9::csplit), which leaves room for five CTAs per SM.
// Threads own fixed positions k = t + 256 m of the colour sub-lattice, which
// are also the shared-memory indices inside a colour plane.
//
// k_resid_restrict<VAR>: r = b - A x on the fine nodes of a coarse tile (x and
// coefficients staged the same way), then rc = R r with R = P^T
// (multigrid.cpp:120-123); also zeroes the coarse iterate.
#include "kernels.hpp"

namespace ocb {

std::atomic<int> g_sweep_lean{1}; // operands of variable sweeps read in the passes (see SweepShape); 1 measured best (C4 P_T -3%)

namespace {

// words per node record of the colour-split copy: 8 off-diagonals (SW, S, SE, W,
// E, NW, N, NE), 1/a_ii, one pad word (records stay 16-byte aligned)
constexpr int kRecW = 10;

__device__ __forceinline__ void cp_async8(void* dst_smem, const void* src)
{
    const unsigned s = (unsigned)__cvta_generic_to_shared(dst_smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all()
{
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
}

// (P ec)(gx, gy): bilinear prolongation, parents in ascending column order,
// branch-free (weight 0 = absent parent; no local-memory arrays)
__device__ __forceinline__ double prolong_at2(const double* __restrict__ ec, int nxc, int gx, int gy)
{
    int x0, x1, y0, y1;
    double wx0, wx1, wy0, wy1;
    if (gx & 1) {
        x0 = x1 = (gx - 1) >> 1;
        wx0 = 1.0;
        wx1 = 0.0;
    } else {
        x0 = gx / 2 - 1;
        x1 = gx / 2;
        wx0 = x0 >= 0 ? 0.5 : 0.0;
        wx1 = x1 < nxc ? 0.5 : 0.0;
    }
    if (gy & 1) {
        y0 = y1 = (gy - 1) >> 1;
        wy0 = 1.0;
        wy1 = 0.0;
    } else {
        y0 = gy / 2 - 1;
        y1 = gy / 2;
        wy0 = y0 >= 0 ? 0.5 : 0.0;
        wy1 = y1 < nxc ? 0.5 : 0.0;
    }
    double e = 0.0;
    if (wy0 != 0.0) {
        const double* r = ec + (long long)y0 * nxc;
        if (wx0 != 0.0) e += (wx0 * wy0) * r[x0];
        if (wx1 != 0.0) e += (wx1 * wy0) * r[x1];
    }
    if (wy1 != 0.0) {
        const double* r = ec + (long long)y1 * nxc;
        if (wx0 != 0.0) e += (wx0 * wy1) * r[x0];
        if (wx1 != 0.0) e += (wx1 * wy1) * r[x1];
    }
    return e;
}

// MODE 0: plain; 1: + divergence check (one more updated ring); 2: + residual
// and restriction (two more updated rings). Extra rings are staged in pairs so
// the region origin stays even.
// LEAN (variable operators read through L1 only): 1 = 1/a_ii, 2 = 1/a_ii and b are
// read from global memory in the passes instead of being staged (smaller
// footprint, more CTAs per SM: the passes are load-latency bound).
template <int TX, int TY, int NS, bool VAR, int MODE = 0, int LEAN_ = 0>
struct SweepShape {
    static constexpr int H = 4 * NS + (MODE ? 2 : 0);
    static constexpr int RX = TX + 2 * H, RY = TY + 2 * H;
    static constexpr int R = RX * RY;
    // Shared-memory layout: colour-planar. Plane c = (lx & 1) + 2 (ly & 1) holds
    // the region nodes of one colour, row-major over the colour sub-lattice
    // (CXN x CYN), so a colour pass reads every operand at unit stride (the
    // natural layout reads every other word: two-way bank conflicts on each
    // 64-bit access). The plane stride is padded to 8 mod 16 words so the
    // staging copies (lanes alternate between two planes) stay conflict-free.
    static constexpr int CXN = RX / 2, CYN = RY / 2, KC = CXN * CYN;
    static constexpr int PS = KC + (24 - KC % 16) % 16;
    static constexpr int RP = 4 * PS; // words per staged field
    // variable coefficients are staged in shared memory whenever the 11 planes
    // fit (coalesced row copies, read once per launch for all fused sweeps);
    // otherwise read through L1 (colour-strided, L2-bandwidth bound)
    static constexpr bool CS = VAR && (size_t)11 * RP * sizeof(double) <= 100 * 1024; // >= 2 CTAs/SM
    // LEAN_ = 3 (RING): a producer warp streams each colour pass's node records
    // (Op9::csplit, one bulk copy per colour row: the TMA engine's 1-D copies,
    // completion on an mbarrier) into a two-stage ring two passes ahead of the
    // 256 compute threads, which then read coefficients and 1/a_ii from shared
    // memory instead of waiting on L2 in every pass.
    static constexpr bool RING = VAR && !CS && LEAN_ == 3 &&
                                 ((size_t)2 * RP + 2 * KC * kRecW + (MODE == 2 ? (TX + 1) * (TY + 1) : 0)) * sizeof(double) <=
                                     112 * 1024; // two CTAs per SM, else the in-pass loads (LEAN 1)
    static constexpr int LEAN = (VAR && !CS) ? (RING ? 1 : LEAN_) : 0;
    static constexpr int PLANES = CS ? 11 : 3 - LEAN; // x, b, inv (+ 8 off-diagonals)
    static constexpr int RINGW = RING ? 2 * KC * kRecW : 0; // two stages of KC records
    static constexpr int THREADS = RING ? 288 : 256;
    static constexpr int RSX = TX + 1, RSN = (TX + 1) * (TY + 1); // MODE 2: fine residual rows
    static constexpr size_t smem = ((size_t)PLANES * RP + RINGW + (MODE == 2 ? RSN : 0)) * sizeof(double);
    // planar index of region node (lx, ly)
    __host__ __device__ static constexpr int pidx(int lx, int ly)
    {
        return ((lx & 1) + 2 * (ly & 1)) * PS + (ly >> 1) * CXN + (lx >> 1);
    }
};

// RN: the last sweeps of a V-cycle also run MgHierarchy::solve's divergence
// check (multigrid.cpp:141-157): the final pass updates one ring beyond the
// tile, so the tile's residual b - A x is exact in shared memory; its squares
// are summed per CTA and the last CTA applies finish_norm_check.
struct NormCheck {
    double* part;
    unsigned* counter;
    double* state;
    int* flags;
};
// MODE 2: the last pre-smoothing launch of a level also computes bc = R (b - A x)
// for the coarse nodes whose centre fine node lies in its tile (zeroing xc),
// as k_resid_restrict does: the final pass updates two rings beyond the tile.
struct RestrictOut {
    double* bc;
    double* xc;
};

__device__ __forceinline__ void ring_wait(unsigned bar, unsigned parity)
{
    asm volatile(
        "{\n .reg .pred p;\n RW:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra RW;\n}" ::"r"(bar),
        "r"(parity)
        : "memory");
}

template <int TX, int TY, int NS, bool VAR, int MODE = 0, int LEAN_ = 0>
__global__ void __launch_bounds__(SweepShape<TX, TY, NS, VAR, MODE, LEAN_>::THREADS) k_sweep(Op9 A, const double* __restrict__ b,
                                               const double* __restrict__ inv,
                                               const double* __restrict__ xin,
                                               double* __restrict__ xout,
                                               const double* __restrict__ ec, int forward,
                                               int zero_init, NormCheck nc, RestrictOut ro)
{
    constexpr bool RN = MODE == 1, RR = MODE == 2;
    using S = SweepShape<TX, TY, NS, VAR, MODE, LEAN_>;
    constexpr int H = S::H, RX = S::RX, RY = S::RY, RP = S::RP, PS = S::PS, LEAN = S::LEAN;
    constexpr bool RING = S::RING;
    constexpr int P = 4 * NS;
    extern __shared__ double sm[];
    double* xs = sm;
    double* bs = xs + RP;
    double* iv = bs + RP;
    double* cs = iv + RP; // VAR: plane p holds entry d = p < 4 ? p : p + 1
    double* ring = sm + S::PLANES * RP; // RING: two stages of node records
    __shared__ unsigned long long ring_bar[2];
    const bool comp = !RING || threadIdx.x < 256; // RING: warp 8 is the producer
    if (RING && threadIdx.x == 0) {
        const unsigned b0 = (unsigned)__cvta_generic_to_shared(&ring_bar[0]);
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\nmbarrier.init.shared::cta.b64 [%1], 1;\n"
                     "fence.mbarrier_init.release.cluster;\n" ::"r"(b0), "r"(b0 + 8)
                     : "memory");
    }

    const int nx = A.nx;
    const long long n = (long long)nx * nx;
    const int nxc = (nx - 1) / 2;
    const int tx0 = blockIdx.x * TX, ty0 = blockIdx.y * TY;
    const int ox = tx0 - H, oy = ty0 - H;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;

    // ---- stage the region: every copy in flight before the first wait
    for (int ly = comp ? ty : RY; ly < RY; ly += 8) {
        const int gy = oy + ly;
        const bool rowin = gy >= 0 && gy < nx;
        for (int lx = tx; lx < RX; lx += 32) {
            const int gx = ox + lx;
            const int l = S::pidx(lx, ly);
            if (rowin && gx >= 0 && gx < nx) {
                const long long i = (long long)gy * nx + gx;
                if (zero_init) xs[l] = 0.0;
                else cp_async8(xs + l, xin + i);
                if (LEAN < 2) cp_async8(bs + l, b + i);
                if (LEAN < 1) cp_async8(iv + l, inv + i);
                if (S::CS) {
#pragma unroll
                    for (int p = 0; p < 8; ++p) cp_async8(cs + p * RP + l, A.coef + (p < 4 ? p : p + 1) * n + i);
                }
            } else {
                xs[l] = 0.0;
                if (LEAN < 2) bs[l] = 0.0;
                if (LEAN < 1) iv[l] = 0.0;
                if (S::CS) {
#pragma unroll
                    for (int p = 0; p < 8; ++p) cs[p * RP + l] = 0.0;
                }
            }
        }
    }
    cp_async_wait_all();
    if (ec) {
        __syncthreads();
        for (int ly = comp ? ty : RY; ly < RY; ly += 8) {
            const int gy = oy + ly;
            if (gy < 0 || gy >= nx) continue;
            for (int lx = tx; lx < RX; lx += 32) {
                const int gx = ox + lx;
                if (gx < 0 || gx >= nx) continue;
                const int l = S::pidx(lx, ly);
                xs[l] = xs[l] + prolong_at2(ec, nxc, gx, gy); // x += P ec
            }
        }
    }
    __syncthreads();

    // Fixed node table: thread t owns colour-sub-lattice positions k = t + 256 m
    // of the region (region origin ox, oy is even, so a colour's nodes are
    // (2 kx + cx, 2 ky + cy) in region coordinates for every pass). k is also
    // the node's index inside its colour plane; the neighbours of a colour-c
    // node sit at pass-uniform offsets from k in the other planes.
    constexpr int CXN = S::CXN, KC = S::KC, KT = (KC + 255) / 256;
    static_assert(RX % 2 == 0 && RY % 2 == 0, "even regions keep colour parity");
    int kx0[KT], ky0[KT], ks0[KT];
#pragma unroll
    for (int m = 0; m < KT; ++m) {
        const int k = threadIdx.x + 256 * m;
        const int ky = k / CXN, kx = k - ky * CXN;
        kx0[m] = k < KC ? ox + 2 * kx : -(1 << 30); // out-of-range marker
        ky0[m] = oy + 2 * ky;
        ks0[m] = ky0[m] * nx + (ox >> 1) + kx; // colour-split node index less the pass offset
    }
    long long cpo[9]; // coefficient plane offsets d * n (variable operators)
#pragma unroll
    for (int d = 0; d < 9; ++d) cpo[d] = (long long)d * n;
    // RING producer: the records of pass q's colour rows, one bulk copy per row
    // (lane = colour row), into stage q & 1; bytes complete on that stage's mbarrier
    auto produce = [&](int q) {
        const int pc = q & 3;
        const int c = forward ? pc : 3 - pc;
        const int cx = c & 1, cy = c >> 1;
        const int g = P - 1 - q + (RN ? 1 : 0) + (RR ? 2 : 0);
        const int lox = max(tx0 - g, 0), hix = min(tx0 + TX + g, nx);
        const int loy = max(ty0 - g, 0), hiy = min(ty0 + TY + g, nx);
        const unsigned bar = (unsigned)__cvta_generic_to_shared(&ring_bar[q & 1]);
        double* stg = ring + (q & 1) * (S::KC * kRecW);
        const int lane = threadIdx.x & 31;
        const int gy = oy + 2 * lane + cy;
        if (lane < S::CYN && gy >= loy && gy < hiy) {
            const int k0 = (lox - ox - cx + 1) >> 1;    // first and last colour column in range
            const int k1 = (hix - 1 - ox - cx) >> 1;
            if (k1 >= k0) {
                const unsigned bytes = (unsigned)(k1 - k0 + 1) * kRecW * 8u;
                const double* src = A.csplit + ((long long)gy * nx + (cx ? ((nx + 1) >> 1) : 0) + (ox >> 1) + k0) * kRecW;
                const unsigned dst = (unsigned)__cvta_generic_to_shared(stg + (lane * S::CXN + k0) * kRecW);
                asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
                             "l"(src), "r"(bytes), "r"(bar)
                             : "memory");
            }
        }
        __syncwarp();
        if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
    };
    if (RING && !comp) {
        produce(0);
        produce(1);
    }
#pragma unroll 1
    for (int q = 0; q < P; ++q) {
        const int pc = q & 3;
        const int c = forward ? pc : 3 - pc;
        const int cx = c & 1, cy = c >> 1;
        const int g = P - 1 - q + (RN ? 1 : 0) + (RR ? 2 : 0);
        const int lox = max(tx0 - g, 0), hix = min(tx0 + TX + g, nx);
        const int loy = max(ty0 - g, 0), hiy = min(ty0 + TY + g, nx);
        const int lc = c * PS;
        const int so = cy * nx + (cx ? ((nx + 1) >> 1) : 0); // colour-split index offset of this pass
        int off[9]; // neighbour d of a colour-c node k: xs[off[d] + k]
#pragma unroll
        for (int d = 0; d < 9; ++d) {
            const int dx = d % 3 - 1, dy = d / 3 - 1;
            const int ncx = dx ? cx ^ 1 : cx, ncy = dy ? cy ^ 1 : cy;
            const int sx = dx < 0 ? cx - 1 : (dx > 0 ? cx : 0); // sub-lattice column shift
            const int sy = dy < 0 ? cy - 1 : (dy > 0 ? cy : 0);
            off[d] = (ncx + 2 * ncy) * PS + sy * CXN + sx;
        }
        if (RING) {
            if (comp) {
                ring_wait((unsigned)__cvta_generic_to_shared(&ring_bar[q & 1]), (unsigned)(q >> 1) & 1u);
                const double2* stg = reinterpret_cast<const double2*>(ring + (q & 1) * (S::KC * kRecW));
#pragma unroll
                for (int m = 0; m < KT; ++m) {
                    const int gx = kx0[m] + cx, gy = ky0[m] + cy;
                    if (gx >= lox && gx < hix && gy >= loy && gy < hiy) {
                        const int k = threadIdx.x + 256 * m;
                        const int l = lc + k;
                        const double2* rec = stg + k * (kRecW / 2);
                        const double2 a01 = rec[0], a23 = rec[1], a45 = rec[2], a67 = rec[3];
                        const double ivl = rec[4].x;
                        double s = bs[l];
                        s -= a01.x * xs[off[0] + k];
                        s -= a01.y * xs[off[1] + k];
                        s -= a23.x * xs[off[2] + k];
                        s -= a23.y * xs[off[3] + k];
                        s -= a45.x * xs[off[5] + k];
                        s -= a45.y * xs[off[6] + k];
                        s -= a67.x * xs[off[7] + k];
                        s -= a67.y * xs[off[8] + k];
                        xs[l] = s * ivl;
                    }
                }
            }
            __syncthreads(); // pass q done: its stage is free
            if (!comp && q + 2 < P) produce(q + 2);
            continue;
        }
#pragma unroll
        for (int m = 0; m < KT; ++m) {
            const int gx = kx0[m] + cx, gy = ky0[m] + cy;
            if (gx >= lox && gx < hix && gy >= loy && gy < hiy) {
                const int k = threadIdx.x + 256 * m;
                const int l = lc + k;
                const double* cp = VAR ? A.coef + ((long long)gy * nx + gx) : nullptr;
                const long long gi = (long long)gy * nx + gx;
                double s = LEAN == 2 ? __ldg(b + gi) : bs[l];
                if (VAR && !S::CS && A.csplit) {
                    // the node's record: 8 off-diagonals in four 16-byte loads
                    const int si = ks0[m] + so;
                    const double2* rec = reinterpret_cast<const double2*>(A.csplit) + (long long)si * (kRecW / 2);
                    const double2 a01 = __ldg(rec), a23 = __ldg(rec + 1), a45 = __ldg(rec + 2),
                                  a67 = __ldg(rec + 3);
                    const double ivl = LEAN >= 1 ? __ldg(reinterpret_cast<const double*>(rec + 4)) : iv[l];
                    s -= a01.x * xs[off[0] + k];
                    s -= a01.y * xs[off[1] + k];
                    s -= a23.x * xs[off[2] + k];
                    s -= a23.y * xs[off[3] + k];
                    s -= a45.x * xs[off[5] + k];
                    s -= a45.y * xs[off[6] + k];
                    s -= a67.x * xs[off[7] + k];
                    s -= a67.y * xs[off[8] + k];
                    xs[l] = s * ivl;
                    continue;
                }
                const double ivl = LEAN >= 1 ? __ldg(inv + gi) : iv[l];
#pragma unroll
                for (int d = 0; d < 9; ++d) {
                    if (d == 4) continue;
                    double a;
                    if (S::CS) a = cs[(d < 4 ? d : d - 1) * RP + l];
                    else if (VAR) a = __ldg(cp + cpo[d]);
                    else a = A.c[d];
                    s -= a * xs[off[d] + k];
                }
                xs[l] = s * ivl;
            }
        }
        __syncthreads();
    }

    double acc = 0.0;
    for (int ly = comp ? ty : TY; ly < TY; ly += 8) {
        const int gy = ty0 + ly;
        if (gy >= nx) break;
        for (int lx = tx; lx < TX; lx += 32) {
            const int gx = tx0 + lx;
            if (gx >= nx) continue;
            const int l = S::pidx(lx + H, ly + H);
            const long long i = (long long)gy * nx + gx;
            xout[i] = xs[l];
            if (RN) { // r = b - A x in the reference's row order (op_apply_at)
                double sum = 0.0;
#pragma unroll
                for (int d = 0; d < 9; ++d) {
                    double a = VAR ? __ldg(A.coef + cpo[d] + i) : A.c[d];
                    if (d == 4 && A.diag) a += __ldg(A.diag + i);
                    sum += a * xs[S::pidx(lx + H + (d % 3 - 1), ly + H + (d / 3 - 1))];
                }
                const double r = (LEAN == 2 ? __ldg(b + i) : bs[l]) - sum;
                acc += r * r;
            }
        }
    }
    if (RN) {
        __shared__ double red[32];
        acc = block_sum(acc, red);
        if (threadIdx.x == 0) nc.part[blockIdx.y * gridDim.x + blockIdx.x] = acc;
        finish_norm_check(nc.part, nc.counter, nc.state, nc.flags, 0);
    }
    if (RR) {
        // fine residual on [tx0, tx0+TX] x [ty0, ty0+TY] (multigrid.cpp:120-121,
        // k_resid_restrict's order), then R = P^T for this tile's coarse nodes
        double* rs = sm + S::PLANES * RP + S::RINGW;
        for (int ly = comp ? ty : TY + 1; ly <= TY; ly += 8) {
            const int gy = ty0 + ly;
            for (int lx = tx; lx <= TX; lx += 32) {
                const int gx = tx0 + lx;
                double r = 0.0;
                if (gx < nx && gy < nx) {
                    const long long i = (long long)gy * nx + gx;
                    double sum = 0.0;
#pragma unroll
                    for (int d = 0; d < 9; ++d) {
                        double a = VAR ? __ldg(A.coef + cpo[d] + i) : A.c[d];
                        if (d == 4 && A.diag) a += __ldg(A.diag + i);
                        sum += a * xs[S::pidx(lx + H + (d % 3 - 1), ly + H + (d / 3 - 1))];
                    }
                    r = (LEAN == 2 ? __ldg(b + i) : bs[S::pidx(lx + H, ly + H)]) - sum;
                }
                rs[ly * S::RSX + lx] = r;
            }
        }
        __syncthreads();
        const int cx0 = tx0 / 2, cy0 = ty0 / 2;
        for (int j = comp ? ty : TY; j < TY / 2; j += 8) {
            const int cy = cy0 + j;
            for (int kx = tx; kx < TX / 2; kx += 32) {
                const int cx = cx0 + kx;
                if (cx >= nxc || cy >= nxc) continue;
                double sum = 0.0;
#pragma unroll
                for (int a = 0; a < 3; ++a) {
                    const double wy = (a == 1) ? 1.0 : 0.5;
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        const double wx = (c == 1) ? 1.0 : 0.5;
                        sum += (wx * wy) * rs[(2 * j + a) * S::RSX + 2 * kx + c];
                    }
                }
                const long long I = (long long)cy * nxc + cx;
                ro.bc[I] = sum;
                if (ro.xc) ro.xc[I] = 0.0;
            }
        }
    }
}

// r = b - A x on the fine tile of a CX x CY coarse tile, then R = P^T.
template <int CX, int CY, bool VAR>
__global__ void __launch_bounds__(256) k_resid_restrict(Op9 A, const double* __restrict__ b,
                                                        const double* __restrict__ x,
                                                        double* __restrict__ bc,
                                                        double* __restrict__ xc)
{
    constexpr int FX = 2 * CX + 1, FY = 2 * CY + 1; // fine nodes feeding the coarse tile
    constexpr int XX = FX + 2, XY = FY + 2;         // plus the stencil halo
    constexpr int F = FX * FY;
    extern __shared__ double sm[];
    double* xs = sm;            // XX*XY
    double* rs = xs + XX * XY;  // F (b on entry, r after)
    double* cf = rs + F;        // VAR: 9*F coefficients
    const int nx = A.nx;
    const long long n = (long long)nx * nx;
    const int nxc = (nx - 1) / 2;
    const int cx0 = blockIdx.x * CX, cy0 = blockIdx.y * CY;
    const int fx0 = 2 * cx0, fy0 = 2 * cy0;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    for (int ly = ty; ly < XY; ly += 8) {
        const int gy = fy0 - 1 + ly;
        for (int lx = tx; lx < XX; lx += 32) {
            const int gx = fx0 - 1 + lx;
            if (gx >= 0 && gx < nx && gy >= 0 && gy < nx) cp_async8(xs + ly * XX + lx, x + (long long)gy * nx + gx);
            else xs[ly * XX + lx] = 0.0;
        }
    }
    for (int ly = ty; ly < FY; ly += 8) {
        const int gy = fy0 + ly;
        for (int lx = tx; lx < FX; lx += 32) {
            const int gx = fx0 + lx;
            const int l = ly * FX + lx;
            if (gx < nx && gy < nx) {
                const long long i = (long long)gy * nx + gx;
                cp_async8(rs + l, b + i);
                if (VAR) {
#pragma unroll
                    for (int d = 0; d < 9; ++d) cp_async8(cf + d * F + l, A.coef + d * n + i);
                }
            } else {
                rs[l] = 0.0;
                if (VAR) {
#pragma unroll
                    for (int d = 0; d < 9; ++d) cf[d * F + l] = 0.0;
                }
            }
        }
    }
    cp_async_wait_all();
    __syncthreads();
    for (int ly = ty; ly < FY; ly += 8) {
        const int gy = fy0 + ly;
        for (int lx = tx; lx < FX; lx += 32) {
            const int gx = fx0 + lx;
            const int l = ly * FX + lx;
            if (gx < nx && gy < nx) {
                const int lxs = (ly + 1) * XX + lx + 1;
                double s = 0.0; // multigrid.cpp:120-121: r = A x; r = rhs - r
#pragma unroll
                for (int d = 0; d < 9; ++d) {
                    double a = VAR ? cf[d * F + l] : A.c[d];
                    if (d == 4 && A.diag) a += A.diag[(long long)gy * nx + gx];
                    s += a * xs[lxs + (d / 3 - 1) * XX + (d % 3 - 1)];
                }
                rs[l] = rs[l] - s;
            }
        }
    }
    __syncthreads();
    for (int j = ty; j < CY; j += 8) {
        const int cy = cy0 + j;
        for (int k = tx; k < CX; k += 32) {
            const int cx = cx0 + k;
            if (cx >= nxc || cy >= nxc) continue;
            double s = 0.0;
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                const double wy = (a == 1) ? 1.0 : 0.5;
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    const double wx = (c == 1) ? 1.0 : 0.5;
                    s += (wx * wy) * rs[(2 * j + a) * FX + 2 * k + c];
                }
            }
            const long long I = (long long)cy * nxc + cx;
            bc[I] = s;
            if (xc) xc[I] = 0.0;
        }
    }
}

// colour-split copy of a variable operator for the tiled sweep: row y holds its
// even-x nodes, then its odd-x nodes, so one colour pass reads consecutive
// node records: the 8 off-diagonals of a node next to each other (four 16-byte
// loads from one address instead of eight strided planes), and 1/a_ii
// (k_inv_diag's quotient) in the same node order
__global__ void k_colour_split(int nx, const double* __restrict__ coef, const double* __restrict__ diag,
                               double* __restrict__ out)
{
    const long long n = (long long)nx * nx;
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int gy = (int)(i / nx), gx = (int)(i - (long long)gy * nx);
    const long long o = (long long)gy * nx + ((gx & 1) ? ((nx + 1) >> 1) + (gx >> 1) : (gx >> 1));
    const int p = blockIdx.y;
    if (p < 8) {
        out[o * kRecW + p] = coef[(p < 4 ? p : p + 1) * n + i];
    } else {
        double a = coef[4 * n + i];
        if (diag) a += diag[i];
        out[o * kRecW + 8] = 1.0 / a;
        out[o * kRecW + 9] = 0.0;
    }
}

__global__ void k_inv_diag(Op9 A, double* __restrict__ inv, long long fcs, long long fds,
                           double* __restrict__ dfull)
{
    const long long n = (long long)A.nx * A.nx;
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int bt = blockIdx.y;
    double a = A.coef ? A.coef[bt * fcs + 4 * n + i] : A.c[4];
    if (A.diag) a += A.diag[bt * fds + i];
    inv[bt * n + i] = 1.0 / a;
    if (dfull) dfull[bt * n + i] = a;
}

template <int TX, int TY, int NS, bool VAR, int MODE, int LEAN = 0>
void sweep_go_lean(cudaStream_t s, const Op9& A, const double* b, const double* inv, const double* x,
                   double* xo, bool forward, bool zero_init, const double* ec, const NormCheck& nc,
                   const RestrictOut& ro)
{
    constexpr size_t smem = SweepShape<TX, TY, NS, VAR, MODE, LEAN>::smem;
    static const bool attr = [] { // thread-safe one-time setup
        cudaFuncSetAttribute(k_sweep<TX, TY, NS, VAR, MODE, LEAN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
        return true;
    }();
    (void)attr;
    dim3 grid((A.nx + TX - 1) / TX, (A.nx + TY - 1) / TY);
    note_launch();
    k_sweep<TX, TY, NS, VAR, MODE, LEAN><<<grid, SweepShape<TX, TY, NS, VAR, MODE, LEAN>::THREADS, smem, s>>>(
        A, b, inv, x, xo, ec, forward ? 1 : 0, zero_init ? 1 : 0, nc, ro);
}

template <int TX, int TY, int NS, bool VAR, int MODE>
void sweep_go_mode(cudaStream_t s, const Op9& A, const double* b, const double* inv, const double* x,
                   double* xo, bool forward, bool zero_init, const double* ec, const NormCheck& nc,
                   const RestrictOut& ro)
{
    if constexpr (VAR && !SweepShape<TX, TY, NS, VAR, MODE>::CS && NS <= 2) {
        const int lean = g_sweep_lean.load();
        if (lean == 3 && A.csplit) return sweep_go_lean<TX, TY, NS, VAR, MODE, 3>(s, A, b, inv, x, xo, forward, zero_init, ec, nc, ro);
        if (lean == 1 || lean == 3) return sweep_go_lean<TX, TY, NS, VAR, MODE, 1>(s, A, b, inv, x, xo, forward, zero_init, ec, nc, ro);
        if (lean == 2) return sweep_go_lean<TX, TY, NS, VAR, MODE, 2>(s, A, b, inv, x, xo, forward, zero_init, ec, nc, ro);
    }
    sweep_go_lean<TX, TY, NS, VAR, MODE, 0>(s, A, b, inv, x, xo, forward, zero_init, ec, nc, ro);
}

// the fused variants only for the 1- and 2-sweep launches that end a phase
template <int TX, int TY, int NS, bool VAR>
void sweep_go(cudaStream_t s, const Op9& A, const double* b, const double* inv, const double* x,
              double* xo, bool forward, bool zero_init, const double* ec, const NormCheck* nc,
              const RestrictOut* ro)
{
    if constexpr (NS <= 2) {
        if (nc) {
            sweep_go_mode<TX, TY, NS, VAR, 1>(s, A, b, inv, x, xo, forward, zero_init, ec, *nc, RestrictOut{});
            return;
        }
        if (ro) {
            sweep_go_mode<TX, TY, NS, VAR, 2>(s, A, b, inv, x, xo, forward, zero_init, ec, NormCheck{}, *ro);
            return;
        }
    }
    sweep_go_mode<TX, TY, NS, VAR, 0>(s, A, b, inv, x, xo, forward, zero_init, ec, NormCheck{}, RestrictOut{});
}

template <int TX, int TY, int NS>
void sweep_pick_var(cudaStream_t s, const Op9& A, const double* b, const double* inv,
                    const double* x, double* xo, bool forward, bool zero_init, const double* ec,
                    const NormCheck* nc, const RestrictOut* ro)
{
    if (A.coef) sweep_go<TX, TY, NS, true>(s, A, b, inv, x, xo, forward, zero_init, ec, nc, ro);
    else sweep_go<TX, TY, NS, false>(s, A, b, inv, x, xo, forward, zero_init, ec, nc, ro);
}

template <int NS>
void sweep_tile(int id, cudaStream_t s, const Op9& A, const double* b, const double* inv,
                const double* x, double* xo, bool forward, bool zero_init, const double* ec,
                const NormCheck* nc, const RestrictOut* ro)
{
    switch (id) {
    case 0:
        if constexpr (NS <= 2) {
            sweep_go<64, 32, NS, false>(s, A, b, inv, x, xo, forward, zero_init, ec, nc, ro);
            break;
        }
        [[fallthrough]];
    case 1: sweep_pick_var<32, 32, NS>(s, A, b, inv, x, xo, forward, zero_init, ec, nc, ro); break;
    case 2: sweep_pick_var<32, 16, NS>(s, A, b, inv, x, xo, forward, zero_init, ec, nc, ro); break;
    case 4:
        if constexpr (NS <= 2) {
            sweep_pick_var<32, 24, NS>(s, A, b, inv, x, xo, forward, zero_init, ec, nc, ro);
            break;
        }
        sweep_pick_var<32, 32, NS>(s, A, b, inv, x, xo, forward, zero_init, ec, nc, ro);
        break;
    default: sweep_pick_var<16, 16, NS>(s, A, b, inv, x, xo, forward, zero_init, ec, nc, ro); break;
    }
}

} // namespace

std::atomic<int> g_cluster_bottom{1};
std::atomic<int> g_cluster_top8{1};
std::atomic<int> g_sweep_tile{-1}; // tuning override: -1 auto, else tile id (see launch_sweep_tiled)
std::atomic<int> g_sweep_fuse{2};  // sweeps fused per launch (measured best, profiles/r01/tuning.md)

std::atomic<int> g_colour_split{1};
std::atomic<int> g_fuse_norm{1};
std::atomic<int> g_fuse_restrict{1};

void launch_colour_split(cudaStream_t s, int nx, const double* coef, const double* diag, double* out)
{
    const long long n = (long long)nx * nx;
    note_launch();
    k_colour_split<<<dim3((unsigned)((n + 255) / 256), 9), 256, 0, s>>>(nx, coef, diag, out);
}

void launch_inv_diag(cudaStream_t s, const Op9& A, double* inv, int batch, long long fcs,
                     long long fds, double* dfull)
{
    const long long n = (long long)A.nx * A.nx;
    note_launch();
    k_inv_diag<<<dim3((unsigned)((n + 255) / 256), batch), 256, 0, s>>>(A, inv, fcs, fds, dfull);
}

bool launch_sweep_tiled(cudaStream_t s, const Op9& A, const double* b, const double* inv,
                        const double* x, double* xo, bool forward, bool zero_init,
                        const double* ec, int ns, double* part, unsigned* counter, double* state,
                        int* flags, double* bc, double* xc)
{
    int id = g_sweep_tile;
    if (id < 0) {
        // Alone on the GPU a sweep is latency-bound: prefer more, smaller tiles.
        // With several solves in flight (one context each) the sweeps compete
        // for bandwidth: prefer the larger tiles (less halo re-read).
        const bool shared = active_contexts() > 1;
        // variable 1023^2 levels: 32x24 tiles = 1376 CTAs = 1.86 waves of the 740
        // resident CTAs (32x32: 1024 = 1.38 waves, a second round 38% full)
        if (A.nx >= 1000) id = A.coef ? 4 : 1;
        else if (A.nx >= 500) id = shared ? (A.coef ? 1 : 0) : 2;
        else id = (shared && A.coef) ? 1 : 3;
    }
    if (id == 0 && (A.coef || ns > 2)) id = 1; // 64x32 tiles: constant stencils, <= 2 sweeps
    // fuse the divergence check when asked for, the launch sweeps <= 2 times and
    // its grid fits the partials buffer (kNormBlocks)
    const int T = id == 0 ? 64 : 32, TYy = id == 0 ? 32 : (id == 1 ? 32 : (id == 4 ? 24 : 16));
    const int TXx = id == 3 ? 16 : T;
    const long long nb = (long long)((A.nx + TXx - 1) / TXx) * ((A.nx + TYy - 1) / TYy);
    NormCheck nc{part, counter, state, flags};
    const NormCheck* pnc = (part && ns <= 2 && nb <= kNormBlocks) ? &nc : nullptr;
    RestrictOut ro{bc, xc};
    const RestrictOut* pro = (!pnc && bc && ns <= 2) ? &ro : nullptr;
    switch (ns) {
    case 1: sweep_tile<1>(id, s, A, b, inv, x, xo, forward, zero_init, ec, pnc, pro); break;
    case 2: sweep_tile<2>(id, s, A, b, inv, x, xo, forward, zero_init, ec, pnc, pro); break;
    case 3: sweep_tile<3>(id, s, A, b, inv, x, xo, forward, zero_init, ec, nullptr, nullptr); break;
    case 4: sweep_tile<4>(id, s, A, b, inv, x, xo, forward, zero_init, ec, nullptr, nullptr); break;
    default: sweep_tile<5>(id, s, A, b, inv, x, xo, forward, zero_init, ec, nullptr, nullptr); break;
    }
    return pnc != nullptr || pro != nullptr;
}

void launch_resid_restrict_tiled(cudaStream_t s, const Op9& A, const double* b, const double* x,
                                 double* bc, double* xc)
{
    constexpr int CX = 32, CY = 8;
    constexpr int F = (2 * CX + 1) * (2 * CY + 1);
    constexpr int XS = (2 * CX + 3) * (2 * CY + 3);
    const int nxc = (A.nx - 1) / 2;
    dim3 grid((nxc + CX - 1) / CX, (nxc + CY - 1) / CY);
    note_launch();
    if (A.coef) {
        constexpr size_t smem = (size_t)(XS + 10 * F) * sizeof(double);
        static const bool attr = [] { // thread-safe one-time setup
            cudaFuncSetAttribute(k_resid_restrict<CX, CY, true>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            return true;
        }();
        (void)attr;
        k_resid_restrict<CX, CY, true><<<grid, 256, smem, s>>>(A, b, x, bc, xc);
    } else {
        constexpr size_t smem = (size_t)(XS + F) * sizeof(double);
        k_resid_restrict<CX, CY, false><<<grid, 256, smem, s>>>(A, b, x, bc, xc);
    }
}

} // namespace ocb
