// Saddle-operator and preconditioner-block kernels (sm_100a, FP64).
//
// Each kernel is one pass over the grid with the 9-point stencils applied
// matrix-free (constant L, M, M+tau L) or from 9 coefficient arrays (SUPG
// convection-diffusion, partial observation mass). Arithmetic follows the
// reference's evaluation order term by term so results agree to rounding.
#include "kernels.hpp"

#include <algorithm>

namespace ocb {

namespace {

constexpr int kT = 256;

inline unsigned blocks_for(long long n) { return (unsigned)((n + kT - 1) / kT); }

__device__ __forceinline__ double stencil_diff(const Op9& A, const double* __restrict__ w,
                                               const double* __restrict__ v, int gx, int gy)
{
    // (A (w - v))_i with the difference formed per entry first (qp.cpp:84-87)
    const int nx = A.nx;
    const long long n = (long long)nx * nx;
    const long long i = (long long)gy * nx + gx;
    double s = 0.0;
#pragma unroll
    for (int d = 0; d < 9; ++d) {
        const int jx = gx + d % 3 - 1, jy = gy + d / 3 - 1;
        if (jx < 0 || jx >= nx || jy < 0 || jy >= nx) continue;
        const long long j = (long long)jy * nx + jx;
        s += op_coef(A, d, i, n) * (w[j] - v[j]);
    }
    return s;
}

// ---------------------------------------------------------------- KKT (steady)
// make_saddle_operator (ipm.cpp:244-267) over steady_matvecs (ipm.cpp:347-374):
//   ry = (M_obs y + th_y y) + L^T p
//   rw = (alpha M(w-v) + th_w w) - M p
//   rv = (alpha (-M(w-v)) + th_v v) + M p
//   rp = L y - M(w-v)
template <bool HAS_TY, bool RESID>
__global__ void __launch_bounds__(kT) k_kkt_steady(ProbDev P, const double* __restrict__ ty,
                                                   const double* __restrict__ tw,
                                                   const double* __restrict__ tv,
                                                   const double* __restrict__ x,
                                                   double* __restrict__ out,
                                                   const double* __restrict__ b,
                                                   double* __restrict__ part)
{
    __shared__ double sh[32];
    const long long n = P.ns;
    const int nx = P.nx;
    const double* y = x;
    const double* w = x + n;
    const double* v = x + 2 * n;
    const double* p = x + 3 * n;
    double acc = 0.0;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const int ii = (int)i, gy = ii / nx, gx = ii - gy * nx; // 32-bit: n < 2^31
        const double My = op_apply_at(P.Mobs, y, gx, gy);
        const double Ltp = op_apply_at(P.LT, p, gx, gy);
        const double Mwv = stencil_diff(P.M, w, v, gx, gy);
        const double Mp = op_apply_at(P.M, p, gx, gy);
        const double Ly = op_apply_at(P.L, y, gx, gy);
        double ry = My;
        if (HAS_TY) ry += ty[i] * y[i];
        ry = ry + Ltp;
        const double rw = (P.alpha * Mwv + tw[i] * w[i]) - Mp;
        const double rv = (P.alpha * (-Mwv) + tv[i] * v[i]) + Mp;
        const double rp = Ly - Mwv;
        if (RESID) {
            const double d0 = b[i] - ry, d1 = b[n + i] - rw, d2 = b[2 * n + i] - rv,
                         d3 = b[3 * n + i] - rp;
            acc += d0 * d0 + d1 * d1 + d2 * d2 + d3 * d3;
        }
        if (out) {
            out[i] = ry;
            out[n + i] = rw;
            out[2 * n + i] = rv;
            out[3 * n + i] = rp;
        }
    }
    if (RESID) {
        acc = block_sum(acc, sh);
        if (threadIdx.x == 0) part[blockIdx.x] = acc;
    }
}

// ---------------------------------------------------- KKT (steady), tiled
// The same operator and arithmetic as k_kkt_steady (each stencil sum in the
// reference's entry order, one FMA per entry), staged through shared memory:
// a CTA handles 32 x 16 node tiles; y, p and the difference w - v of the tile
// plus a one-node halo are loaded once with coalesced row loads (positions
// outside the grid hold 0, which adds nothing to a sum: fma(a, 0, s) = s), so
// every field word is read from DRAM about once (1.2x with the halo) instead
// of nine times through L1. 256 threads, two nodes each (rows ty, ty + 8);
// the coefficient arrays of variable operators (SUPG L, L^T, partial M_obs)
// are read per node, coalesced along the tile rows. RESID: the fixed grid of
// kRedBlocks CTAs walks the tiles in a fixed order, so the block partials of
// |b - A x|^2 are deterministic.
constexpr int kKX = 32, kKY = 16, kKH = kKX + 2, kKV = kKY + 2;

__device__ __forceinline__ double op_tile_at(const Op9& A, const double* __restrict__ s, int sx,
                                             int sy, int i, int n)
{
    // s: tile of the field (pitch kKH) with a one-node halo; (sx, sy) = tile
    // position of the node (halo-shifted), i = its global index
    double acc = 0.0;
#pragma unroll
    for (int d = 0; d < 9; ++d) {
        double a = A.coef ? A.coef[d * n + i] : A.c[d];
        if (d == 4 && A.diag) a += A.diag[i];
        acc += a * s[(sy + d / 3 - 1) * kKH + sx + d % 3 - 1];
    }
    return acc;
}

template <bool HAS_TY, bool RESID>
__global__ void __launch_bounds__(256) k_kkt_tiled(ProbDev P, const double* __restrict__ ty,
                                                   const double* __restrict__ tw,
                                                   const double* __restrict__ tv,
                                                   const double* __restrict__ x,
                                                   double* __restrict__ out,
                                                   const double* __restrict__ b,
                                                   double* __restrict__ part)
{
    __shared__ double sy_[kKV * kKH], sp_[kKV * kKH], sd_[kKV * kKH];
    __shared__ double sh[32];
    const int nx = P.nx;
    const int n = nx * nx; // < 2^31
    const double* y = x;
    const double* w = x + n;
    const double* v = x + 2 * (long long)n;
    const double* p = x + 3 * (long long)n;
    const int tilesx = (nx + kKX - 1) / kKX, tilesy = (nx + kKY - 1) / kKY;
    const int ntiles = tilesx * tilesy;
    const int tx = threadIdx.x & 31, tyy = threadIdx.x >> 5; // 8 warps
    double acc = 0.0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int x0 = (t % tilesx) * kKX, y0 = (t / tilesx) * kKY;
        __syncthreads(); // the previous tile's readers are done
        // halo tiles: warp r loads rows r, r + 8, ... (34 columns: lanes 0..31, then 32..33)
        for (int r = tyy; r < kKV; r += 8) {
            const int gy = y0 + r - 1;
            const bool rok = gy >= 0 && gy < nx;
#pragma unroll
            for (int c0 = 0; c0 < kKH; c0 += 32) {
                const int c = c0 + tx;
                if (c < kKH) {
                    const int gx = x0 + c - 1;
                    const bool ok = rok && gx >= 0 && gx < nx;
                    const int i = ok ? gy * nx + gx : 0;
                    sy_[r * kKH + c] = ok ? __ldcs(y + i) : 0.0;
                    sp_[r * kKH + c] = ok ? __ldcs(p + i) : 0.0;
                    sd_[r * kKH + c] = ok ? __ldcs(w + i) - __ldcs(v + i) : 0.0;
                }
            }
        }
        __syncthreads();
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int ly = tyy + 8 * h;
            const int gx = x0 + tx, gy = y0 + ly;
            if (gx >= nx || gy >= nx) continue;
            const int i = gy * nx + gx;
            const int sx = tx + 1, sy = ly + 1;
            const double yi = sy_[sy * kKH + sx];
            const double pi = sp_[sy * kKH + sx];
            const double My = op_tile_at(P.Mobs, sy_, sx, sy, i, n);
            const double Ltp = op_tile_at(P.LT, sp_, sx, sy, i, n);
            const double Mwv = op_tile_at(P.M, sd_, sx, sy, i, n);
            const double Mp = op_tile_at(P.M, sp_, sx, sy, i, n);
            const double Ly = op_tile_at(P.L, sy_, sx, sy, i, n);
            double ry = My;
            if (HAS_TY) ry += ty[i] * yi;
            ry = ry + Ltp;
            const double wi = __ldcs(w + i), vi = __ldcs(v + i);
            const double rw = (P.alpha * Mwv + tw[i] * wi) - Mp;
            const double rv = (P.alpha * (-Mwv) + tv[i] * vi) + Mp;
            const double rp = Ly - Mwv;
            if (RESID) {
                const double d0 = b[i] - ry, d1 = b[n + i] - rw, d2 = b[2 * (long long)n + i] - rv,
                             d3 = b[3 * (long long)n + i] - rp;
                acc += d0 * d0 + d1 * d1 + d2 * d2 + d3 * d3;
            }
            if (out) {
                __stcs(out + i, ry);
                __stcs(out + n + i, rw);
                __stcs(out + 2 * (long long)n + i, rv);
                __stcs(out + 3 * (long long)n + i, rp);
            }
        }
    }
    if (RESID) {
        acc = block_sum(acc, sh);
        if (threadIdx.x == 0) part[blockIdx.x] = acc;
    }
}

// ------------------------------------------------------------------ KKT (heat)
// space-time blocks (timedep.cpp:18-133), block k of ns nodes, s_k = tau w_k:
//   hy = s_k (M y_k);  K y = Mtl y_k - M y_{k-1};  K^T p = Mtl p_k - M p_{k+1}
//   hz = [a_k M(w-v); -a_k M(w-v)], a_k = alpha tau w_k;  B z = tau (M(w-v))
//   B^T p = [tau (M p); -tau (M p)]
template <bool HAS_TY, bool RESID>
__global__ void __launch_bounds__(kT) k_kkt_heat(ProbDev P, const double* __restrict__ ty,
                                                 const double* __restrict__ tw,
                                                 const double* __restrict__ tv,
                                                 const double* __restrict__ x,
                                                 double* __restrict__ out,
                                                 const double* __restrict__ b,
                                                 double* __restrict__ part)
{
    __shared__ double sh[32];
    const long long ns = P.ns, N = P.ny;
    const int nx = P.nx;
    const double* y = x;
    const double* w = x + N;
    const double* v = x + 2 * N;
    const double* p = x + 3 * N;
    double acc = 0.0;
    for (long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x; g < N;
         g += (long long)gridDim.x * blockDim.x) {
        const int k = (int)g / (int)ns; // 32-bit: the space-time size is < 2^31
        const long long i = g - (long long)k * ns;
        const int ii = (int)i, gy = ii / nx, gx = ii - gy * nx; // 32-bit: n < 2^31
        const long long off = (long long)k * ns;
        const double sk = P.tau * P.qw[k];
        const double ak = P.alpha * P.tau * P.qw[k];
        const double hy = sk * op_apply_at(P.M, y + off, gx, gy);
        double ktp = op_apply_at(P.Mtl, p + off, gx, gy);
        if (k + 1 < P.nt) ktp -= op_apply_at(P.M, p + off + ns, gx, gy);
        double ky = op_apply_at(P.Mtl, y + off, gx, gy);
        if (k > 0) ky -= op_apply_at(P.M, y + off - ns, gx, gy);
        const double Mwv = stencil_diff(P.M, w + off, v + off, gx, gy);
        const double Mp = op_apply_at(P.M, p + off, gx, gy);
        double ry = hy;
        if (HAS_TY) ry += ty[g] * y[g];
        ry = ry + ktp;
        const double rw = (ak * Mwv + tw[g] * w[g]) - P.tau * Mp;
        const double rv = ((-ak) * Mwv + tv[g] * v[g]) + P.tau * Mp;
        const double rp = ky - P.tau * Mwv;
        if (RESID) {
            const double d0 = b[g] - ry, d1 = b[N + g] - rw, d2 = b[2 * N + g] - rv,
                         d3 = b[3 * N + g] - rp;
            acc += d0 * d0 + d1 * d1 + d2 * d2 + d3 * d3;
        }
        if (out) {
            out[g] = ry;
            out[N + g] = rw;
            out[2 * N + g] = rv;
            out[3 * N + g] = rp;
        }
    }
    if (RESID) {
        acc = block_sum(acc, sh);
        if (threadIdx.x == 0) part[blockIdx.x] = acc;
    }
}

// ------------------------------------------------------------ KKT (heat), tiled
// The same operator and arithmetic as k_kkt_heat (every stencil sum in the
// reference's entry order, one FMA per entry), staged through shared memory:
// a CTA handles one 32 x 16 node tile of one time block k. y_k, y_{k-1}, p_k,
// p_{k+1} and the difference w_k - v_k of the tile plus a one-node halo are
// loaded once with coalesced row loads (0 outside the grid and for the absent
// neighbour blocks: fma(a, 0, s) = s, and the k-edge terms are skipped as in
// k_kkt_heat), instead of 54 loads per node through L1. A thread owns two
// vertically adjacent nodes and reads each field's 4 x 3 window once (30
// shared loads per node). Tiles are numbered time-fastest, so the CTAs that
// share y_k / p_k tiles run together and the re-read hits L2. RESID: the
// fixed grid of kRedBlocks CTAs walks the tiles in a fixed order
// (deterministic partials of |b - A x|^2).
// The RESID launch has 512 threads: two independent 256-thread halves, each
// walking its own tiles with its own named barrier, so the fixed grid still
// keeps four tile pipelines per SM in flight.
template <bool HAS_TY, bool RESID>
__global__ void __launch_bounds__(RESID ? 512 : 256) k_kkt_heat_tiled(ProbDev P, const double* __restrict__ ty,
                                                        const double* __restrict__ tw,
                                                        const double* __restrict__ tv,
                                                        const double* __restrict__ x,
                                                        double* __restrict__ out,
                                                        const double* __restrict__ b,
                                                        double* __restrict__ part)
{
    constexpr int T = kKV * kKH;
    extern __shared__ double kkt_sm[];
    const int half = RESID ? (threadIdx.x >> 8) : 0;
    double* sf = kkt_sm + half * 5 * T; // y_k, y_{k-1}, p_k, p_{k+1}, w_k - v_k
    __shared__ double sh[32];
    auto half_sync = [&]() {
        if (RESID) asm volatile("bar.sync %0, 256;" ::"r"(1 + half) : "memory");
        else __syncthreads();
    };
    const int nx = P.nx, nt = P.nt;
    const long long ns = P.ns, N = P.ny;
    const double* y = x;
    const double* w = x + N;
    const double* v = x + 2 * N;
    const double* p = x + 3 * N;
    const int tilesx = (nx + kKX - 1) / kKX, tilesy = (nx + kKY - 1) / kKY;
    const long long ntiles = (long long)tilesx * tilesy * nt;
    const int tx = threadIdx.x & 31, tyy = (threadIdx.x >> 5) & 7; // 8 warps per tile
    double acc = 0.0;
    const long long tstep = RESID ? 2LL * gridDim.x : gridDim.x;
    for (long long t = RESID ? 2LL * blockIdx.x + half : blockIdx.x; t < ntiles; t += tstep) {
        const int k = (int)(t % nt);
        const int ts = (int)(t / nt);
        const int x0 = (ts % tilesx) * kKX, y0 = (ts / tilesx) * kKY;
        const long long off = (long long)k * ns;
        const bool hm = k > 0, hp = k + 1 < nt;
        half_sync(); // the previous tile's readers are done
        for (int r = tyy; r < kKV; r += 8) {
            const int gy = y0 + r - 1;
            const bool rok = gy >= 0 && gy < nx;
#pragma unroll
            for (int c0 = 0; c0 < kKH; c0 += 32) {
                const int c = c0 + tx;
                if (c < kKH) {
                    const int gx = x0 + c - 1;
                    const bool ok = rok && gx >= 0 && gx < nx;
                    const long long i = ok ? off + (long long)gy * nx + gx : 0;
                    const int l = r * kKH + c;
                    sf[l] = ok ? __ldg(y + i) : 0.0;
                    sf[T + l] = (ok && hm) ? __ldg(y + i - ns) : 0.0;
                    sf[2 * T + l] = ok ? __ldg(p + i) : 0.0;
                    sf[3 * T + l] = (ok && hp) ? __ldg(p + i + ns) : 0.0;
                    sf[4 * T + l] = ok ? __ldcs(w + i) - __ldcs(v + i) : 0.0;
                }
            }
        }
        half_sync();
        const int gx = x0 + tx;
        const int ly = 2 * tyy; // rows ly, ly + 1 of the tile
        if (gx < nx && y0 + ly < nx) {
            // stencil sums of the two nodes from a field's 4 x 3 window, in
            // op_apply_at's entry order (d = 0..8, one FMA per entry)
            double My[2], Mly[2], Mym[2], Mp[2], Mlp[2], Mpp[2], Mwv[2];
            auto window = [&](const double* f, double (&q)[12]) {
#pragma unroll
                for (int rr = 0; rr < 4; ++rr)
#pragma unroll
                    for (int cc = 0; cc < 3; ++cc) q[rr * 3 + cc] = f[(ly + rr) * kKH + tx + cc];
            };
            auto sum9 = [&](const double (&c)[9], const double (&q)[12], int h) {
                double a = 0.0;
#pragma unroll
                for (int d = 0; d < 9; ++d) a += c[d] * q[h * 3 + d];
                return a;
            };
            {
                double q[12];
                window(sf, q);
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    My[h] = sum9(P.M.c, q, h);
                    Mly[h] = sum9(P.Mtl.c, q, h);
                }
                window(sf + T, q);
#pragma unroll
                for (int h = 0; h < 2; ++h) Mym[h] = sum9(P.M.c, q, h);
                window(sf + 2 * T, q);
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    Mlp[h] = sum9(P.Mtl.c, q, h);
                    Mp[h] = sum9(P.M.c, q, h);
                }
                window(sf + 3 * T, q);
#pragma unroll
                for (int h = 0; h < 2; ++h) Mpp[h] = sum9(P.M.c, q, h);
                window(sf + 4 * T, q);
#pragma unroll
                for (int h = 0; h < 2; ++h) Mwv[h] = sum9(P.M.c, q, h);
            }
            const double sk = P.tau * P.qw[k];
            const double ak = P.alpha * P.tau * P.qw[k];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int gy = y0 + ly + h;
                if (gy >= nx) continue;
                const long long g = off + (long long)gy * nx + gx;
                const double hy = sk * My[h];
                double ktp = Mlp[h];
                if (hp) ktp -= Mpp[h];
                double ky = Mly[h];
                if (hm) ky -= Mym[h];
                double ry = hy;
                if (HAS_TY) ry += ty[g] * sf[(ly + h + 1) * kKH + tx + 1];
                ry = ry + ktp;
                const double rw = (ak * Mwv[h] + tw[g] * __ldcs(w + g)) - P.tau * Mp[h];
                const double rv = ((-ak) * Mwv[h] + tv[g] * __ldcs(v + g)) + P.tau * Mp[h];
                const double rp = ky - P.tau * Mwv[h];
                if (RESID) {
                    const double d0 = b[g] - ry, d1 = b[N + g] - rw, d2 = b[2 * N + g] - rv,
                                 d3 = b[3 * N + g] - rp;
                    acc += d0 * d0 + d1 * d1 + d2 * d2 + d3 * d3;
                }
                if (out) {
                    __stcs(out + g, ry);
                    __stcs(out + N + g, rw);
                    __stcs(out + 2 * N + g, rv);
                    __stcs(out + 3 * N + g, rp);
                }
            }
        }
    }
    if (RESID) {
        acc = block_sum(acc, sh);
        if (threadIdx.x == 0) part[blockIdx.x] = acc;
    }
}

// ------------------------------------------------------------------- Chebyshev
// ChebyshevSemiIteration (chebyshev.cpp:9-75) on s_k M + diag(e), Jacobi
// scaled with the fixed interval [1/4, 9/4]: omega = 0.8, rho = 0.8.
__device__ __forceinline__ double cheb_invd(const ProbDev& P, const double* e, int k, long long g)
{
    const double sk = P.heat ? P.tau * P.qw[k] : 1.0;
    const double di = sk * P.M.c[4] + (e ? e[g] : 0.0);
    return 1.0 / di;
}

__global__ void k_cheb_init(ProbDev P, const double* __restrict__ b, const double* __restrict__ e,
                            double omega, double* __restrict__ g_out)
{
    const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= P.ny) return;
    const int k = ((int)g / (int)P.ns);
    g_out[g] = omega * cheb_invd(P, e, k, g) * b[g];
}

__global__ void k_cheb_step(ProbDev P, const double* __restrict__ e, double omega, double wk,
                            const double* __restrict__ prev, const double* __restrict__ cur,
                            const double* __restrict__ gv, double* __restrict__ next)
{
    const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= P.ny) return;
    const long long ns = P.ns;
    const int k = ((int)g / (int)ns);
    const long long i = g - (long long)k * ns;
    const int gy = (int)i / P.nx, gx = (int)i - gy * P.nx; // 32-bit
    double az = op_apply_at(P.M, cur + (long long)k * ns, gx, gy);
    if (P.heat) az = (P.tau * P.qw[k]) * az; // matvec: scale only when scale != 1
    if (e) az += e[g] * cur[g];
    const double invd = cheb_invd(P, e, k, g);
    const double s_cur = cur[g] - omega * invd * az;
    const double pv = prev ? prev[g] : 0.0;
    next[g] = wk * (s_cur + gv[g] - pv) + pv;
}

// Up to kChebTS Chebyshev steps in one launch (temporal blocking): a CTA
// stages the previous two iterates, g and e over its 32x32 tile plus a halo of
// kChebTS nodes in shared memory and advances the region (shrinking by one
// ring per step) in place, the update being k_cheb_step's expressions in the
// same order (cells outside the domain hold 0, as op_apply_at's predicated
// loads read): results equal the step-by-step launches bit for bit. Writes
// the last two iterates of the tile.
constexpr int kChebTS = 5, kChebT = 32, kChebR = kChebT + 2 * kChebTS;
struct ChebSteps {
    double wk[kChebTS];
    int st0, nst; // first step index (>= 2) and steps in this launch
};

// Thread mapping: thread t owns the kChebSeg vertically consecutive region
// nodes of column t % R in row segment t / R, so one 3-column window of
// kChebSeg + 2 rows serves all its stencil sums of a step (27 shared loads for
// 7 nodes instead of 63), and its nodes' g, e and 1/d stay in registers for
// all steps (d as k_cheb_step forms it; no division per step). Only the two
// iterates live in shared memory (one zero row above and below the region).
constexpr int kChebSeg = 7;
static_assert(kChebR % kChebSeg == 0 && (kChebR / kChebSeg) * kChebR <= 256, "column segments cover the region");

__global__ void __launch_bounds__(256, 3) k_cheb_block(ProbDev P, const double* __restrict__ e, double omega,
                                                    ChebSteps S, const double* __restrict__ prev,
                                                    const double* __restrict__ cur,
                                                    const double* __restrict__ gv,
                                                    double* __restrict__ out_prev,
                                                    double* __restrict__ out_cur)
{
    constexpr int R = kChebR, RA = (R + 2) * R, SEG = kChebSeg;
    extern __shared__ double csm[];
    double* pa = csm + R;      // previous iterate (row -1 and row R are zero rows)
    double* pc = pa + RA;      // current iterate
    const int nx = P.nx, k = blockIdx.z;
    const long long off = (long long)k * P.ns;
    const int tx0 = blockIdx.x * kChebT, ty0 = blockIdx.y * kChebT;
    const int ox = tx0 - kChebTS, oy = ty0 - kChebTS;
    const int cx = threadIdx.x % R, r0 = (threadIdx.x / R) * SEG;
    const bool own = threadIdx.x < (R / SEG) * R;
    const int gx = ox + cx;
    for (int l = threadIdx.x; l < R; l += blockDim.x) { // zero rows
        csm[l] = 0.0;
        csm[RA + l] = 0.0;
        csm[(R + 1) * R + l] = 0.0;
        csm[RA + (R + 1) * R + l] = 0.0;
    }
    const double sk = P.heat ? P.tau * P.qw[k] : 1.0;
    double gr[SEG], er[SEG], idr[SEG];
    bool in[SEG];
    if (own) {
#pragma unroll
        for (int m = 0; m < SEG; ++m) {
            const int gy = oy + r0 + m;
            in[m] = gx >= 0 && gx < nx && gy >= 0 && gy < nx;
            double a = 0.0, c = 0.0;
            gr[m] = er[m] = 0.0;
            if (in[m]) {
                const long long g = off + (long long)gy * nx + gx;
                a = prev ? prev[g] : 0.0;
                c = cur[g];
                gr[m] = gv[g];
                er[m] = e ? e[g] : 0.0;
            }
            idr[m] = 1.0 / (sk * P.M.c[4] + (e ? er[m] : 0.0));
            pa[(r0 + m) * R + cx] = a;
            pc[(r0 + m) * R + cx] = c;
        }
    }
    __syncthreads();
    for (int i = 0; i < S.nst; ++i) {
        const int st = S.st0 + i;
        const double wk = S.wk[i];
        const int lo = i + 1, hi = R - i - 1; // region rows/columns still exact after this step
        if (own && cx >= lo && cx < hi) {
            // rolling window: rows r0+m-1 .. r0+m+1, columns cx-1 .. cx+1 of the current iterate
            double q[9];
#pragma unroll
            for (int rr = 0; rr < 2; ++rr)
#pragma unroll
                for (int cc = 0; cc < 3; ++cc) q[(rr + 1) * 3 + cc] = pc[(r0 + rr - 1) * R + cx + cc - 1];
#pragma unroll
            for (int m = 0; m < SEG; ++m) {
#pragma unroll
                for (int cc = 0; cc < 3; ++cc) {
                    q[cc] = q[3 + cc];
                    q[3 + cc] = q[6 + cc];
                    q[6 + cc] = pc[(r0 + m + 1) * R + cx + cc - 1];
                }
                const int ly = r0 + m;
                if (ly < lo || ly >= hi || !in[m]) continue;
                // k_cheb_step's expressions with the contractions it compiles to
                // spelled out (the hoisted omega / d product must not change them)
                double az = 0.0;
#pragma unroll
                for (int d = 0; d < 9; ++d) az = __fma_rn(P.M.c[d], q[d], az);
                if (P.heat) az = __dmul_rn(__dmul_rn(P.tau, P.qw[k]), az);
                const double pcl = q[4];
                if (e) az = __fma_rn(er[m], pcl, az);
                const double s_cur = __fma_rn(az, __dmul_rn(omega, -idr[m]), pcl);
                const int l = ly * R + cx;
                const double pv = st == 2 ? 0.0 : pa[l];
                pa[l] = __fma_rn(wk, __dsub_rn(__dadd_rn(s_cur, gr[m]), pv), pv);
            }
        }
        __syncthreads();
        double* t = pa;
        pa = pc;
        pc = t;
    }
    if (own && cx >= kChebTS && cx < kChebTS + kChebT && gx < nx) {
#pragma unroll
        for (int m = 0; m < SEG; ++m) {
            const int ly = r0 + m, gy = oy + ly;
            if (ly < kChebTS || ly >= kChebTS + kChebT || gy >= nx) continue;
            const long long g = off + (long long)gy * nx + gx;
            if (out_prev) out_prev[g] = pa[ly * R + cx];
            out_cur[g] = pc[ly * R + cx];
        }
    }
}

// ------------------------------------------------------------------ 2x2 block
__global__ void k_control_2x2(ProbDev P, const double* __restrict__ tw,
                              const double* __restrict__ tv, const double* __restrict__ rw,
                              const double* __restrict__ rv, double* __restrict__ vw,
                              double* __restrict__ vv, int* flags)
{
    const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= P.ny) return;
    const int k = ((int)g / (int)P.ns);
    const double dM = P.M.c[4];
    const double sc = P.heat ? P.alpha * P.tau * P.qw[k] : P.alpha;
    const double a = sc * dM + tw[g];
    const double bb = -sc * dM;
    const double c = sc * dM + tv[g];
    if (a == 0.0) { atomicOr(flags, kErrSingular2x2); return; }
    const double schur = c - bb * bb / a;
    if (schur == 0.0) { atomicOr(flags, kErrSingular2x2); return; }
    const double x2 = (rv[g] - bb * rw[g] / a) / schur;
    const double x1 = (rw[g] - bb * x2) / a;
    vw[g] = x1;
    vv[g] = x2;
}

// -------------------------------------------------------------- coupling rows
__global__ void k_coupling_steady(ProbDev P, const double* __restrict__ vy,
                                  const double* __restrict__ vw, const double* __restrict__ vv,
                                  const double* __restrict__ rp, double* __restrict__ t)
{
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= P.ns) return;
    const int gy = (int)i / P.nx, gx = (int)i - gy * P.nx; // 32-bit
    const double Lvy = op_apply_at(P.L, vy, gx, gy);
    const double mw = op_apply_at(P.M, vw, gx, gy);
    const double mv = op_apply_at(P.M, vv, gx, gy);
    t[i] = Lvy + ((-mw + mv) - rp[i]);
}

__global__ void k_coupling_heat(ProbDev P, const double* __restrict__ vy,
                                const double* __restrict__ vw, const double* __restrict__ vv,
                                const double* __restrict__ rp, double* __restrict__ t)
{
    const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= P.ny) return;
    const long long ns = P.ns;
    const int k = ((int)g / (int)ns);
    const long long i = g - (long long)k * ns;
    const long long off = (long long)k * ns;
    const int gy = (int)i / P.nx, gx = (int)i - gy * P.nx; // 32-bit
    double ly = op_apply_at(P.Mtl, vy + off, gx, gy);
    if (k > 0) ly -= op_apply_at(P.M, vy + off - ns, gx, gy);
    const double cz = P.tau * stencil_diff(P.M, vw + off, vv + off, gx, gy);
    t[g] = ly + (-cz - rp[g]);
}

__global__ void k_schur_middle(ProbDev P, const double* __restrict__ ty,
                               const double* __restrict__ t1, double* __restrict__ t2)
{
    const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= P.ny) return;
    const long long ns = P.ns;
    const int k = ((int)g / (int)ns);
    const long long i = g - (long long)k * ns;
    const int gy = (int)i / P.nx, gx = (int)i - gy * P.nx; // 32-bit
    const double tyv = ty ? ty[g] : 0.0;
    if (P.heat) {
        const double m = op_apply_at(P.M, t1 + (long long)k * ns, gx, gy);
        t2[g] = (P.tau * P.qw[k]) * m + tyv * t1[g];
    } else {
        double m = op_apply_at(P.Mobs, t1, gx, gy);
        if (ty) m += tyv * t1[g];
        t2[g] = m;
    }
}

__global__ void k_ppi_rhs1(ProbDev P, const double* __restrict__ vw, const double* __restrict__ vv,
                           const double* __restrict__ rp, double* __restrict__ rhs1)
{
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= P.ns) return;
    const int gy = (int)i / P.nx, gx = (int)i - gy * P.nx; // 32-bit
    rhs1[i] = stencil_diff(P.M, vw, vv, gx, gy) + rp[i];
}

__global__ void k_ppi_t(ProbDev P, const double* __restrict__ ty, const double* __restrict__ v1,
                        const double* __restrict__ ry, double* __restrict__ t)
{
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= P.ns) return;
    const int gy = (int)i / P.nx, gx = (int)i - gy * P.nx; // 32-bit
    const double tyv = ty ? ty[i] : 0.0;
    t[i] = op_apply_at(P.Mobs, v1, gx, gy) + (tyv * v1[i] - ry[i]);
}

__global__ void k_op_apply(Op9 A, const double* __restrict__ x, double* __restrict__ y)
{
    const long long n = (long long)A.nx * A.nx;
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int ii = (int)i, gy = ii / A.nx;
    y[i] = op_apply_at(A, x, ii - gy * A.nx, gy);
}

__global__ void k_rhs_plus_mass(ProbDev P, const double* __restrict__ r,
                                const double* __restrict__ xnb, double* __restrict__ rhs)
{
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= P.ns) return;
    const int gy = (int)i / P.nx, gx = (int)i - gy * P.nx; // 32-bit
    rhs[i] = xnb ? r[i] + op_apply_at(P.M, xnb, gx, gy) : r[i];
}

__global__ void k_mhat(ProbDev P, const double* __restrict__ ty, const double* __restrict__ tw,
                       const double* __restrict__ tv, double* __restrict__ mhat,
                       double* __restrict__ bracket, int* flags)
{
    const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= P.ny) return;
    const double d = P.M.c[4];
    const double twv = tw[g], tvv = tv[g];
    const double tyv = ty ? ty[g] : 0.0;
    if (d <= 0.0 || twv <= 0.0 || tvv <= 0.0 || tyv < 0.0) {
        atomicOr(flags, kErrBadInput);
        return;
    }
    const double s = 1.0 / twv + 1.0 / tvv;
    double br;
    double scale_d;
    if (P.heat) {
        const int k = ((int)g / (int)P.ns);
        const double dc = P.qw[k] * d;
        br = P.tau * P.tau * d * d * s / (P.alpha * P.tau * dc * s + 1.0);
        scale_d = P.tau * dc;
    } else {
        br = d * d * s / (P.alpha * d * s + 1.0);
        scale_d = d;
    }
    if (br < -1e-14) atomicOr(flags, kErrNegBracket);
    br = fmax(br, 0.0);
    if (bracket) bracket[g] = br;
    if (mhat) mhat[g] = sqrt(br) * sqrt(scale_d + tyv);
}

} // namespace

void launch_mhat(cudaStream_t s, const ProbDev& P, const double* ty, const double* tw,
                 const double* tv, double* mhat, double* bracket, int* flags)
{
    note_launch();
    k_mhat<<<blocks_for(P.ny), kT, 0, s>>>(P, ty, tw, tv, mhat, bracket, flags);
}

void launch_kkt(cudaStream_t s, const ProbDev& P, const double* ty, const double* tw,
                const double* tv, const double* x, double* out, const double* b, double* part)
{
    const bool has_ty = ty != nullptr;
    const bool resid = part != nullptr;
    const long long N = P.ny;
    const unsigned grid = resid ? kRedBlocks : blocks_for(N);
    if (P.heat && g_kkt_tiled.load(std::memory_order_relaxed) && !P.M.coef && !P.Mtl.coef &&
        !P.M.diag && !P.Mtl.diag) {
        const long long nt = (long long)((P.nx + kKX - 1) / kKX) * ((P.nx + kKY - 1) / kKY) * P.nt;
        const unsigned g = resid ? kRedBlocks : (unsigned)nt;
        constexpr size_t sm1 = 5 * (size_t)kKV * kKH * sizeof(double);
        static const bool attr = [] { // the two-tile RESID variants exceed the 48 KB default
            cudaFuncSetAttribute(k_kkt_heat_tiled<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(2 * sm1));
            cudaFuncSetAttribute(k_kkt_heat_tiled<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(2 * sm1));
            return true;
        }();
        (void)attr;
        note_launch();
        if (has_ty && resid) k_kkt_heat_tiled<true, true><<<g, 512, 2 * sm1, s>>>(P, ty, tw, tv, x, out, b, part);
        else if (has_ty) k_kkt_heat_tiled<true, false><<<g, 256, sm1, s>>>(P, ty, tw, tv, x, out, b, part);
        else if (resid) k_kkt_heat_tiled<false, true><<<g, 512, 2 * sm1, s>>>(P, ty, tw, tv, x, out, b, part);
        else k_kkt_heat_tiled<false, false><<<g, 256, sm1, s>>>(P, ty, tw, tv, x, out, b, part);
    } else if (P.heat) {
        if (has_ty && resid) { note_launch(); k_kkt_heat<true, true><<<grid, kT, 0, s>>>(P, ty, tw, tv, x, out, b, part); }
        else if (has_ty) { note_launch(); k_kkt_heat<true, false><<<grid, kT, 0, s>>>(P, ty, tw, tv, x, out, b, part); }
        else if (resid) { note_launch(); k_kkt_heat<false, true><<<grid, kT, 0, s>>>(P, ty, tw, tv, x, out, b, part); }
        else { note_launch(); k_kkt_heat<false, false><<<grid, kT, 0, s>>>(P, ty, tw, tv, x, out, b, part); }
    } else if (g_kkt_tiled.load(std::memory_order_relaxed)) {
        // fixed grid for the deterministic residual partials; otherwise one CTA per tile
        const int nt = ((P.nx + kKX - 1) / kKX) * ((P.nx + kKY - 1) / kKY);
        const unsigned g = resid ? kRedBlocks : (unsigned)nt;
        note_launch();
        if (has_ty && resid) k_kkt_tiled<true, true><<<g, 256, 0, s>>>(P, ty, tw, tv, x, out, b, part);
        else if (has_ty) k_kkt_tiled<true, false><<<g, 256, 0, s>>>(P, ty, tw, tv, x, out, b, part);
        else if (resid) k_kkt_tiled<false, true><<<g, 256, 0, s>>>(P, ty, tw, tv, x, out, b, part);
        else k_kkt_tiled<false, false><<<g, 256, 0, s>>>(P, ty, tw, tv, x, out, b, part);
    } else {
        if (has_ty && resid) { note_launch(); k_kkt_steady<true, true><<<grid, kT, 0, s>>>(P, ty, tw, tv, x, out, b, part); }
        else if (has_ty) { note_launch(); k_kkt_steady<true, false><<<grid, kT, 0, s>>>(P, ty, tw, tv, x, out, b, part); }
        else if (resid) { note_launch(); k_kkt_steady<false, true><<<grid, kT, 0, s>>>(P, ty, tw, tv, x, out, b, part); }
        else { note_launch(); k_kkt_steady<false, false><<<grid, kT, 0, s>>>(P, ty, tw, tv, x, out, b, part); }
    }
}

std::atomic<int> g_cheb_block{1};
std::atomic<int> g_kkt_tiled{1};
std::atomic<int> g_heat_fork{1};
std::atomic<int> g_heat_chain{1};
std::atomic<long long> g_tuning_gen{0};

void launch_chebyshev(cudaStream_t s, const ProbDev& P, const double* b, const double* e,
                      int steps, const ChebWork& w, double* out)
{
    const double lmin = 0.25, lmax = 2.25;
    const double omega = 2.0 / (lmin + lmax);
    const double rho = (lmax - lmin) / (lmax + lmin);
    const unsigned grid = blocks_for(P.ny);
    if (steps <= 1) {
        note_launch();
        k_cheb_init<<<grid, kT, 0, s>>>(P, b, e, omega, out);
        return;
    }
    note_launch();
    k_cheb_init<<<grid, kT, 0, s>>>(P, b, e, omega, w.g);
    if (g_cheb_block.load(std::memory_order_relaxed)) {
        // kChebTS steps per launch; the chunks' (previous, current) iterate
        // pairs alternate between (r0, r1) and (r2, out), the last chunk's
        // landing in (r2, out)
        const int nchunk = (steps - 1 + kChebTS - 1) / kChebTS;
        const dim3 bgrid((P.nx + kChebT - 1) / kChebT, (P.nx + kChebT - 1) / kChebT, P.nt);
        const double* prev = nullptr;
        const double* cur = w.g;
        double wk = 1.0;
        int st = 2;
        for (int c = 0; c < nchunk; ++c) {
            const bool pairB = (nchunk - 1 - c) % 2 == 0;
            double* op = pairB ? w.r2 : w.r0;
            double* oc = pairB ? out : w.r1;
            ChebSteps S{};
            S.st0 = st;
            S.nst = std::min(kChebTS, steps - st + 1);
            for (int i = 0; i < S.nst; ++i, ++st) {
                wk = (st == 2) ? 1.0 / (1.0 - 0.5 * rho * rho) : 1.0 / (1.0 - 0.25 * rho * rho * wk);
                S.wk[i] = wk;
            }
            constexpr size_t smem = 2 * (size_t)(kChebR + 2) * kChebR * sizeof(double);
            static const bool attr = cudaFuncSetAttribute(k_cheb_block, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                          (int)smem) == cudaSuccess;
            (void)attr;
            note_launch();
            k_cheb_block<<<bgrid, 256, smem, s>>>(P, e, omega, S, prev, cur, w.g, op, oc);
            prev = op;
            cur = oc;
        }
        return;
    }
    // rotating buffers R[s % 3]; the last step (s = steps) writes into out
    double* R[3] = {w.r0, w.r1, w.r2};
    R[steps % 3] = out;
    double wk = 1.0;
    for (int st = 2; st <= steps; ++st) {
        wk = (st == 2) ? 1.0 / (1.0 - 0.5 * rho * rho) : 1.0 / (1.0 - 0.25 * rho * rho * wk);
        const double* prev = (st == 2) ? nullptr : (st == 3 ? w.g : R[(st - 2) % 3]);
        const double* cur = (st == 2) ? w.g : R[(st - 1) % 3];
        note_launch();
        k_cheb_step<<<grid, kT, 0, s>>>(P, e, omega, wk, prev, cur, w.g, R[st % 3]);
    }
}

void launch_control_2x2(cudaStream_t s, const ProbDev& P, const double* tw, const double* tv,
                        const double* rw, const double* rv, double* vw, double* vv, int* flags)
{
    note_launch();
    k_control_2x2<<<blocks_for(P.ny), kT, 0, s>>>(P, tw, tv, rw, rv, vw, vv, flags);
}

void launch_coupling(cudaStream_t s, const ProbDev& P, const double* vy, const double* vw,
                     const double* vv, const double* rp, double* t)
{
    if (P.heat) { note_launch(); k_coupling_heat<<<blocks_for(P.ny), kT, 0, s>>>(P, vy, vw, vv, rp, t); }
    else { note_launch(); k_coupling_steady<<<blocks_for(P.ns), kT, 0, s>>>(P, vy, vw, vv, rp, t); }
}

void launch_schur_middle(cudaStream_t s, const ProbDev& P, const double* ty, const double* t1,
                         double* t2)
{
    note_launch();
    k_schur_middle<<<blocks_for(P.ny), kT, 0, s>>>(P, ty, t1, t2);
}

void launch_ppi_rhs1(cudaStream_t s, const ProbDev& P, const double* vw, const double* vv,
                     const double* rp, double* rhs1)
{
    note_launch();
    k_ppi_rhs1<<<blocks_for(P.ns), kT, 0, s>>>(P, vw, vv, rp, rhs1);
}

void launch_ppi_t(cudaStream_t s, const ProbDev& P, const double* ty, const double* v1,
                  const double* ry, double* t)
{
    note_launch();
    k_ppi_t<<<blocks_for(P.ns), kT, 0, s>>>(P, ty, v1, ry, t);
}

void launch_op_apply(cudaStream_t s, const Op9& A, const double* x, double* y)
{
    note_launch();
    k_op_apply<<<blocks_for((long long)A.nx * A.nx), kT, 0, s>>>(A, x, y);
}

void launch_rhs_plus_mass(cudaStream_t s, const ProbDev& P, const double* r, const double* xnb,
                          double* rhs)
{
    note_launch();
    k_rhs_plus_mass<<<blocks_for(P.ns), kT, 0, s>>>(P, r, xnb, rhs);
}

} // namespace ocb
