// Geometric multigrid kernels (sm_100a, FP64): prolongation, residual norms
// and the divergence check, Galerkin RAP, coarse LU and the single-CTA bottom
// solver (the tiled sweeps live in k_mg_tiled.cu, the cluster bottom in
// k_mg_cluster.cu, the lexicographic wavefront in k_mg_lex.cu).
//
// Reference semantics (multigrid.cpp):
//   bilinear_prolongation  :10-42   P (1D weights 1/2,1,1/2; Dirichlet dropped), R = P^T
//   gauss_seidel_sweep     :44-66   x_i = (b_i - sum_{j!=i} a_ij x_j) / a_ii
//   MgHierarchy::build     :75-109  Galerkin R A P down to level 2 (or rediscretised base)
//   cycle                  :111-132 pre sweeps, restrict residual, recurse, prolong, post
//   solve                  :141-157 cycles from x=0, throw if ||r|| > 10 ||r_prev||
// Default smoother: 4-colour symmetric Gauss-Seidel (colour = (gx&1) + 2(gy&1),
// forward 0..3 / backward 3..0), the GPU-parallel replacement for the
// lexicographic sweep: it keeps the V-cycle SPD for
// symmetric operators, which MINRES with P_D requires. The lexicographic sweep
// itself is the faithful mode (OC_SMOOTHER_LEX).
#include "kernels.hpp"
#include "lex_gs.cuh"

#include <algorithm>
#include <stdexcept>

namespace ocb {

namespace {

// P row of fine node (gx, gy): coarse parents in ascending column order,
// branch-free (weight 0 = absent parent; no local-memory arrays)
__device__ __forceinline__ double prolong_at(const double* __restrict__ ec, int nxc, int gx, int gy)
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

__device__ __forceinline__ double diag_at(const Op9& A, long long i, long long n)
{
    double a = A.coef ? A.coef[4 * n + i] : A.c[4];
    if (A.diag) a += A.diag[i];
    return a;
}

__global__ void k_prolong_add(int nx, const double* __restrict__ ec, double* __restrict__ x)
{
    const long long n = (long long)nx * nx;
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int ii = (int)i, gy = ii / nx, gx = ii - gy * nx; // 32-bit: n < 2^31
    x[i] = x[i] + prolong_at(ec, (nx - 1) / 2, gx, gy);
}

__global__ void __launch_bounds__(kRedThreads) k_resid_norm_partials(Op9 A,
                                                                     const double* __restrict__ b,
                                                                     const double* __restrict__ x,
                                                                     double* __restrict__ part,
                                                                     unsigned* counter,
                                                                     double* state, int* flags)
{
    __shared__ double sh[32];
    const int nx = A.nx;
    const long long n = (long long)nx * nx;
    double acc = 0.0;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const int ii = (int)i, gy = ii / nx, gx = ii - gy * nx; // 32-bit: n < 2^31
        const double r = b[i] - op_apply_at(A, x, gx, gy);
        acc += r * r;
    }
    acc = block_sum(acc, sh);
    if (threadIdx.x == 0) part[blockIdx.x] = acc;
    finish_norm_check(part, counter, state, flags, 0);
}

__global__ void __launch_bounds__(kRedThreads) k_sq_partials(const double* __restrict__ v,
                                                             long long n, double* __restrict__ part,
                                                             unsigned* counter, double* state)
{
    __shared__ double sh[32];
    double acc = 0.0;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        acc += v[i] * v[i];
    acc = block_sum(acc, sh);
    if (threadIdx.x == 0) part[blockIdx.x] = acc;
    finish_norm_check(part, counter, state, nullptr, 1);
}

// ----------------------------------------------------------------- Galerkin
__device__ __forceinline__ int parents(int g, int nc, int* p, double* w)
{
    if (g & 1) { p[0] = (g - 1) >> 1; w[0] = 1.0; return 1; }
    int k = 0;
    if (g / 2 - 1 >= 0) { p[k] = g / 2 - 1; w[k++] = 0.5; }
    if (g / 2 < nc) { p[k] = g / 2; w[k++] = 0.5; }
    return k;
}

__global__ void k_rap(Op9 A, double* __restrict__ coarse, const double* __restrict__ base,
                      double* __restrict__ rem_out, long long fcs, long long fds, long long ccs)
{
    const int nxf = A.nx, nxc = (nxf - 1) / 2;
    const long long nf = (long long)nxf * nxf, nc = (long long)nxc * nxc;
    const long long C = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (C >= nc) return;
    const int bt = blockIdx.y;
    const double* coef = A.coef ? A.coef + bt * fcs : nullptr;
    const double* dg = A.diag ? A.diag + bt * fds : nullptr;
    const int cx = (int)(C % nxc), cy = (int)(C / nxc);
    double acc[9];
#pragma unroll
    for (int d = 0; d < 9; ++d) acc[d] = 0.0;
    for (int a = 0; a < 3; ++a) {
        const int fy = 2 * cy + a;
        const double wyf = (a == 1) ? 1.0 : 0.5;
        for (int c = 0; c < 3; ++c) {
            const int fx = 2 * cx + c;
            const double wf = ((c == 1) ? 1.0 : 0.5) * wyf;
            const long long fi = (long long)fy * nxf + fx;
            for (int d = 0; d < 9; ++d) {
                const int gx = fx + d % 3 - 1, gy = fy + d / 3 - 1;
                if (gx < 0 || gx >= nxf || gy < 0 || gy >= nxf) continue;
                double av = coef ? coef[d * nf + fi] : A.c[d];
                if (d == 4 && dg) av += dg[fi];
                if (av == 0.0) continue;
                int pxs[2], pys[2];
                double wxs[2], wys[2];
                const int npx = parents(gx, nxc, pxs, wxs), npy = parents(gy, nxc, pys, wys);
                for (int u = 0; u < npy; ++u)
                    for (int v = 0; v < npx; ++v) {
                        const int D = (pys[u] - cy + 1) * 3 + (pxs[v] - cx + 1);
                        acc[D] += wf * av * (wxs[v] * wys[u]);
                    }
            }
        }
    }
    double* out = coarse + bt * ccs;
    // rediscretised levels (multigrid.cpp:94-96): coarse = base + R rem P, and
    // the Galerkin remainder itself is carried to the next level
#pragma unroll
    for (int d = 0; d < 9; ++d) out[d * nc + C] = base ? base[d * nc + C] + acc[d] : acc[d];
    if (rem_out) {
        double* ro = rem_out + bt * ccs;
#pragma unroll
        for (int d = 0; d < 9; ++d) ro[d * nc + C] = acc[d];
    }
}

__global__ void k_remainder9(Op9 A, const double* __restrict__ base, double* __restrict__ rem)
{
    const long long n = (long long)A.nx * A.nx;
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
#pragma unroll
    for (int d = 0; d < 9; ++d) {
        double a = A.coef ? A.coef[d * n + i] : A.c[d];
        if (d == 4 && A.diag) a += A.diag[i];
        rem[d * n + i] = a - base[d * n + i];
    }
}

__global__ void k_coarse_lu(const double* __restrict__ coef9, double* __restrict__ lu,
                            int* __restrict__ perm, long long cstride)
{
    // dense 9x9 from the level-2 (nx = 3) 9-point arrays, column-major
    const int bt = blockIdx.x;
    const double* cf = coef9 + bt * cstride;
    double a[81];
    for (int k = 0; k < 81; ++k) a[k] = 0.0;
    for (int i = 0; i < 9; ++i) {
        const int gx = i % 3, gy = i / 3;
        for (int d = 0; d < 9; ++d) {
            const int jx = gx + d % 3 - 1, jy = gy + d / 3 - 1;
            if (jx < 0 || jx >= 3 || jy < 0 || jy >= 3) continue;
            a[(jy * 3 + jx) * 9 + i] = cf[d * 9 + i];
        }
    }
    int pm[9];
    for (int i = 0; i < 9; ++i) pm[i] = i;
    for (int k = 0; k < 9; ++k) {
        int piv = k;
        double best = fabs(a[k * 9 + k]);
        for (int i = k + 1; i < 9; ++i)
            if (fabs(a[k * 9 + i]) > best) { best = fabs(a[k * 9 + i]); piv = i; }
        if (piv != k) {
            for (int j = 0; j < 9; ++j) {
                const double t = a[j * 9 + k];
                a[j * 9 + k] = a[j * 9 + piv];
                a[j * 9 + piv] = t;
            }
            const int t = pm[k]; pm[k] = pm[piv]; pm[piv] = t;
        }
        const double p = a[k * 9 + k];
        if (p == 0.0) continue;
        for (int i = k + 1; i < 9; ++i) a[k * 9 + i] /= p;
        for (int j = k + 1; j < 9; ++j) {
            const double u = a[j * 9 + k];
            if (u == 0.0) continue;
            for (int i = k + 1; i < 9; ++i) a[j * 9 + i] -= a[k * 9 + i] * u;
        }
    }
    for (int k = 0; k < 81; ++k) lu[bt * 81 + k] = a[k];
    for (int i = 0; i < 9; ++i) perm[bt * 9 + i] = pm[i];
}

// ----------------------------------------------------------- bottom solver
constexpr int kBottomThreads = 1024;

__device__ void bt_sweep(const Op9& A, const double* bsm, double* xsm, bool forward)
{
    const int nx = A.nx;
    const long long n = (long long)nx * nx;
    for (int p = 0; p < 4; ++p) {
        const int c = forward ? p : 3 - p;
        const int cx = c & 1, cy = c >> 1;
        const int cntx = (nx - cx + 1) / 2, cnty = (nx - cy + 1) / 2;
        for (int idx = threadIdx.x; idx < cntx * cnty; idx += blockDim.x) {
            const int gx = cx + 2 * (idx % cntx), gy = cy + 2 * (idx / cntx);
            const long long i = (long long)gy * nx + gx;
            double s = bsm[i];
#pragma unroll
            for (int d = 0; d < 9; ++d) {
                if (d == 4) continue;
                const int jx = gx + d % 3 - 1, jy = gy + d / 3 - 1;
                if (jx < 0 || jx >= nx || jy < 0 || jy >= nx) continue;
                const double a = A.coef ? A.coef[d * n + i] : A.c[d];
                s -= a * xsm[(long long)jy * nx + jx];
            }
            xsm[i] = s / diag_at(A, i, n);
        }
        __syncthreads();
    }
}

// Lexicographic sweep of one bottom level in shared memory (lex_gs.cuh): warps
// 0..ceil(nx/32)-1 run the skewed wavefront; the hand-off between them goes
// through the shared mailbox mbs (sentinel-filled, restored on return). The
// operands of a column (b, old E/NW/N/NE, 1/a_ii from shared memory; the
// coefficients of variable operators from global memory, prefetched into L1)
// are loaded kBtLexR steps ahead into a register ring, so a step's dependent
// chain is the shuffle plus the FMAs of the update.
constexpr int kBtLexR = 4;
constexpr int kBtLexPF = 0; // L1 prefetch distance (0: off)

struct BtRaw {
    double b, e, nw, nn, ne, inv, dd;
    double a[8];
};

__device__ __forceinline__ void bt_lex_load(BtRaw& p, const Op9& A, const double* bsm,
                                            const double* xsm, const double* ism, long long n,
                                            int row0, int sx, int sy, int nx, bool rowok,
                                            bool hasN, bool fwd, int col)
{
    p.b = p.e = p.nw = p.nn = p.ne = p.inv = 0.0;
    p.dd = 1.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) p.a[k] = 0.0;
    if (!rowok || col < 0 || col >= nx) return;
    const int i = row0 + col * sx;
    const bool hasE = col + 1 < nx, hasW = col > 0;
    if (kBtLexPF > 0 && A.coef && col + kBtLexPF < nx) {
#pragma unroll
        for (int d = 0; d < 9; ++d)
            if (d != 4) asm volatile("prefetch.global.L1 [%0];" ::"l"(A.coef + d * n + i + kBtLexPF * sx));
    }
    if (hasE) p.e = xsm[i + sx];
    if (hasN) {
        p.nn = xsm[i + sy];
        if (hasW) p.nw = xsm[i + sy - sx];
        if (hasE) p.ne = xsm[i + sy + sx];
    }
    p.b = bsm[i];
    p.inv = ism[i];
    p.dd = diag_at(A, i, n);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const int d = k < 4 ? k : k + 1;
        const int dp = fwd ? d : 8 - d;
        p.a[k] = A.coef ? __ldg(A.coef + dp * n + i) : A.c[dp];
    }
}

__device__ void bt_sweep_lex(const Op9& A, const double* bsm, double* xsm, const double* ism,
                             volatile double* mbs, bool fwd)
{
    const int nx = A.nx;
    const long long n = (long long)nx * nx;
    const int wid = threadIdx.x >> 5, j = threadIdx.x & 31;
    const int nw = (nx + 31) >> 5;
    if (wid < nw) {
        const int r = 32 * wid + j;
        const bool rowok = r < nx, hasN = r + 1 < nx;
        const int sx = fwd ? 1 : -1, sy = fwd ? nx : -nx;
        const int row0 = fwd ? r * nx : (nx - 1 - r) * nx + (nx - 1);
        const bool consumer = j == 0 && wid > 0, producer = j == 31 && hasN;
        volatile double* mb_in = mbs + (wid > 0 ? wid - 1 : 0) * nx;
        volatile double* mb_out = mbs + wid * nx;
        auto receive = [&](int xe) -> double {
            double v = mb_in[xe];
            while (lex_is_sentinel(v)) v = mb_in[xe];
            mb_in[xe] = lex_sentinel();
            return v;
        };
        double sw = 0.0, s = 0.0, se = 0.0, last = 0.0;
        {   // step -1: lane 0 primes its window with column 0 of row r-1
            double up = __shfl_up_sync(0xffffffffu, last, 1);
            if (j == 0) up = consumer ? receive(0) : 0.0;
            se = up;
        }
        BtRaw ring[kBtLexR];
#pragma unroll
        for (int u = 0; u < kBtLexR; ++u)
            bt_lex_load(ring[u], A, bsm, xsm, ism, n, row0, sx, sy, nx, rowok, hasN, fwd, u - 2 * j);
        const int nsteps = nx + 62;
        for (int base = 0; base < nsteps; base += kBtLexR) {
#pragma unroll
            for (int u = 0; u < kBtLexR; ++u) {
                const int st = base + u;
                const int xl = st - 2 * j;
                const BtRaw& p = ring[u];
                double up = __shfl_up_sync(0xffffffffu, last, 1);
                if (j == 0) {
                    const int xe = st + 1;
                    up = (consumer && xe < nx) ? receive(xe) : 0.0;
                }
                sw = s;
                s = se;
                se = up;
                double v = 0.0;
                if (rowok && xl >= 0 && xl < nx) {
                    // the reference's update (multigrid.cpp:49-60): ascending
                    // physical columns, separate multiply and subtract, s / a_ii
                    v = lex_update_ref(p.a, fwd, p.b, sw, s, se, last, p.e, p.nw, p.nn, p.ne, p.dd,
                                       p.inv);
                    xsm[row0 + xl * sx] = v;
                    if (producer) mb_out[xl] = v;
                }
                last = v;
                bt_lex_load(ring[u], A, bsm, xsm, ism, n, row0, sx, sy, nx, rowok, hasN, fwd,
                            xl + kBtLexR);
            }
        }
    }
    __syncthreads();
}

__device__ double bt_resid_sq(const Op9& A, const double* bsm, const double* xsm, double* red)
{
    const int nx = A.nx;
    double acc = 0.0;
    for (int i = threadIdx.x; i < nx * nx; i += blockDim.x) {
        const double r = bsm[i] - op_apply_at(A, xsm, i % nx, i / nx);
        acc += r * r;
    }
    acc = block_sum(acc, red);
    __syncthreads();
    if (threadIdx.x == 0) red[32] = acc;
    __syncthreads();
    const double out = red[32];
    __syncthreads();
    return out;
}

// LEX: the reference's lexicographic smoother, run by 2 warps as a wavefront
// (64-thread block: registers for the operand rings); else 4-colour, 1024 threads.
template <bool LEX>
__global__ void __launch_bounds__(LEX ? 64 : kBottomThreads)
    k_bottom(BottomArgs a, const double* __restrict__ bg, double* __restrict__ xg, int cycles,
             int pre, int post, int check, double* state, int* flags)
{
    extern __shared__ double sm[];
    __shared__ double red[40];
    double* xs[kBottomMaxLevels];
    double* bs[kBottomMaxLevels];
    double* p = sm;
    for (int k = 0; k < a.nlev; ++k) {
        const int m = a.ops[k].nx * a.ops[k].nx;
        xs[k] = p; p += m;
        bs[k] = p; p += m;
    }
    double* rs = p;
    const int n0 = a.ops[0].nx * a.ops[0].nx;
    volatile double* mbs = rs + n0; // lexicographic hand-off mailbox (64 slots)
    double* is_[kBottomMaxLevels];  // lexicographic mode: 1/a_ii per level
    if (LEX) {
        if (threadIdx.x < 64) mbs[threadIdx.x] = lex_sentinel();
        double* q = rs + n0 + 64;
        for (int k = 0; k < a.nlev; ++k) {
            const Op9& A = a.ops[k];
            const long long m = (long long)A.nx * A.nx;
            is_[k] = q;
            for (int i = threadIdx.x; i < m; i += blockDim.x) q[i] = 1.0 / diag_at(A, i, m);
            q += m;
        }
    }
    for (int i = threadIdx.x; i < n0; i += blockDim.x) {
        bs[0][i] = bg[i];
        xs[0][i] = 0.0;
    }
    __syncthreads();
    double prev = 0.0;
    if (check) {
        double acc = 0.0;
        for (int i = threadIdx.x; i < n0; i += blockDim.x) acc += bs[0][i] * bs[0][i];
        acc = block_sum(acc, red);
        __syncthreads();
        if (threadIdx.x == 0) red[32] = sqrt(acc);
        __syncthreads();
        prev = red[32];
        __syncthreads();
    }
    const int last = a.nlev - 1;
    for (int cyc = 0; cyc < cycles; ++cyc) {
        for (int k = 0; k < last; ++k) {
            const Op9& A = a.ops[k];
            for (int s = 0; s < pre; ++s) {
                if (LEX) bt_sweep_lex(A, bs[k], xs[k], is_[k], mbs, true);
                else bt_sweep(A, bs[k], xs[k], true);
            }
            const int nx = A.nx, nxc = (nx - 1) / 2;
            for (int i = threadIdx.x; i < nx * nx; i += blockDim.x)
                rs[i] = bs[k][i] - op_apply_at(A, xs[k], i % nx, i / nx);
            __syncthreads();
            for (int I = threadIdx.x; I < nxc * nxc; I += blockDim.x) {
                const int cx = I % nxc, cy = I / nxc;
                double s = 0.0;
                for (int u = 0; u < 3; ++u) {
                    const double wy = (u == 1) ? 1.0 : 0.5;
                    for (int v = 0; v < 3; ++v) {
                        const double wx = (v == 1) ? 1.0 : 0.5;
                        s += (wx * wy) * rs[(2 * cy + u) * nx + 2 * cx + v];
                    }
                }
                bs[k + 1][I] = s;
                xs[k + 1][I] = 0.0;
            }
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            // level-2 dense LU solve (DenseFactor::solve)
            double y[9];
            for (int i = 0; i < 9; ++i) y[i] = bs[last][a.perm[i]];
            for (int i = 0; i < 9; ++i)
                for (int k = 0; k < i; ++k) y[i] -= a.lu[k * 9 + i] * y[k];
            for (int i = 8; i >= 0; --i) {
                for (int k = i + 1; k < 9; ++k) y[i] -= a.lu[k * 9 + i] * y[k];
                y[i] /= a.lu[i * 9 + i];
            }
            for (int i = 0; i < 9; ++i) xs[last][i] = y[i];
        }
        __syncthreads();
        for (int k = last - 1; k >= 0; --k) {
            const Op9& A = a.ops[k];
            const int nx = A.nx, nxc = (nx - 1) / 2;
            for (int i = threadIdx.x; i < nx * nx; i += blockDim.x)
                xs[k][i] = xs[k][i] + prolong_at(xs[k + 1], nxc, i % nx, i / nx);
            __syncthreads();
            for (int s = 0; s < post; ++s) {
                if (LEX) bt_sweep_lex(A, bs[k], xs[k], is_[k], mbs, false);
                else bt_sweep(A, bs[k], xs[k], false);
            }
        }
        if (check) {
            const double res = sqrt(bt_resid_sq(a.ops[0], bs[0], xs[0], red));
            if (threadIdx.x == 0 && res > 10.0 * prev) atomicOr(flags, kErrMgDiverged);
            prev = res;
        }
    }
    for (int i = threadIdx.x; i < n0; i += blockDim.x) xg[i] = xs[0][i];
    if (check && threadIdx.x == 0 && state) state[0] = prev;
}

} // namespace

// ------------------------------------------------------------- launchers
void launch_prolong_add(cudaStream_t s, int nx, const double* ec, double* x)
{
    const long long n = (long long)nx * nx;
    note_launch();
    k_prolong_add<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(nx, ec, x);
}

// grid of the fused norm checks: one thread per node up to kNormBlocks blocks
// (fixed per level, so the partial-sum order is deterministic)
static unsigned norm_blocks(long long n)
{
    const long long b = (n + kRedThreads - 1) / kRedThreads;
    return (unsigned)(b < 1 ? 1 : (b > kNormBlocks ? kNormBlocks : b));
}

void launch_residual_norm_check(cudaStream_t s, const Op9& A, const double* b, const double* x,
                                double* part, unsigned* counter, double* state, int* flags)
{
    note_launch();
    k_resid_norm_partials<<<norm_blocks((long long)A.nx * A.nx), kRedThreads, 0, s>>>(
        A, b, x, part, counter, state, flags);
}

void launch_norm_init(cudaStream_t s, const double* b, long long n, double* part,
                      unsigned* counter, double* state)
{
    note_launch();
    k_sq_partials<<<norm_blocks(n), kRedThreads, 0, s>>>(b, n, part, counter, state);
}

void launch_rap(cudaStream_t s, const Op9& fine, double* coarse, const double* base,
                double* rem_out, int batch, long long fcs, long long fds, long long ccs)
{
    const int nxc = (fine.nx - 1) / 2;
    const long long nc = (long long)nxc * nxc;
    dim3 grid((unsigned)((nc + 127) / 128), batch);
    note_launch();
    k_rap<<<grid, 128, 0, s>>>(fine, coarse, base, rem_out, fcs, fds, ccs);
}

void launch_remainder9(cudaStream_t s, const Op9& fine, const double* base9, double* rem9)
{
    const long long n = (long long)fine.nx * fine.nx;
    note_launch();
    k_remainder9<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(fine, base9, rem9);
}

void launch_coarse_lu(cudaStream_t s, const double* coef9, double* lu, int* perm, int batch)
{
    note_launch();
    k_coarse_lu<<<batch, 1, 0, s>>>(coef9, lu, perm, 81);
}

size_t bottom_smem_bytes(const BottomArgs& a)
{
    size_t m = 0;
    for (int k = 0; k < a.nlev; ++k) m += 2ull * a.ops[k].nx * a.ops[k].nx;
    m += (size_t)a.ops[0].nx * a.ops[0].nx;
    m += 64; // lexicographic hand-off mailbox
    if (a.lex)
        for (int k = 0; k < a.nlev; ++k) m += (size_t)a.ops[k].nx * a.ops[k].nx; // 1/a_ii
    return m * sizeof(double);
}

void launch_bottom(cudaStream_t s, const BottomArgs& a, const double* b, double* x, int cycles,
                   int pre, int post, bool check, double* state, int* flags)
{
    const size_t smem = bottom_smem_bytes(a);
    // thread-safe one-time setup (concurrent solves launch from several host threads)
    static const bool attr = [] {
        cudaFuncSetAttribute(k_bottom<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        cudaFuncSetAttribute(k_bottom<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        return true;
    }();
    (void)attr;
    if (smem > 200 * 1024) throw std::runtime_error("bottom solver: level too large for one CTA");
    note_launch();
    if (a.lex)
        k_bottom<true><<<1, 64, smem, s>>>(a, b, x, cycles, pre, post, check ? 1 : 0, state, flags);
    else
        k_bottom<false><<<1, kBottomThreads, smem, s>>>(a, b, x, cycles, pre, post, check ? 1 : 0,
                                                        state, flags);
}

} // namespace ocb
