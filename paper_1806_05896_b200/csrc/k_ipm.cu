// Interior-point step kernels (sm_100a, FP64): barrier diagonals, Newton
// right-hand side, multiplier recovery with fraction-to-boundary min
// reductions, state update with interiority checks, RMS residual norms,
// objective and sparsity. Reference: ipm.cpp:32-235 and 294-329.
#include "kernels.hpp"

namespace ocb {

namespace {

constexpr int kT = 256;
inline unsigned blocks_for(long long n) { return (unsigned)((n + kT - 1) / kT); }

__device__ __forceinline__ double inf_d() { return __longlong_as_double(0x7ff0000000000000LL); }

struct Loc {
    int k;          // time block
    long long i;    // spatial index
    long long off;  // k * ns
    int gx, gy;
};

__device__ __forceinline__ Loc locate(const ProbDev& P, long long g)
{
    Loc l;
    l.k = ((int)g / (int)P.ns);
    l.off = (long long)l.k * P.ns;
    l.i = g - l.off;
    l.gy = (int)l.i / P.nx;
    l.gx = (int)l.i - l.gy * P.nx; // 32-bit: sizes < 2^31
    return l;
}

// (A (x - y))_i with the difference formed per entry
__device__ __forceinline__ double stencil_sub(const Op9& A, const double* __restrict__ x,
                                              const double* __restrict__ y, int gx, int gy)
{
    const int nx = A.nx;
    const long long n = (long long)nx * nx;
    const long long i = (long long)gy * nx + gx;
    double s = 0.0;
#pragma unroll
    for (int d = 0; d < 9; ++d) {
        const int jx = gx + d % 3 - 1, jy = gy + d / 3 - 1;
        if (jx < 0 || jx >= nx || jy < 0 || jy >= nx) continue;
        const long long j = (long long)jy * nx + jx;
        s += op_coef(A, d, i, n) * (x[j] - y[j]);
    }
    return s;
}

// Model block matvecs at one node (steady: ipm.cpp:347-374, heat: timedep.cpp:18-133).
// hz = [hzs*M(w-v); -(hzs*M(w-v))], B z = bs*M(w-v), B^T p = [bs*Mp; -(bs*Mp)].
struct Blocks {
    double hy;     // H_y (y - y_d)
    double ktp;    // K^T p
    double ky;     // K y
    double mwv;    // M (w - v)
    double mp;     // M p
    double hzs;    // alpha (steady) or alpha tau w_k (heat)
    double bs;     // 1 (steady) or tau (heat)
    double bg;     // beta gradient entry (same for the w and v halves)
};

__device__ __forceinline__ Blocks blocks_at(const ProbDev& P, const IpmDev& S, const Loc& l)
{
    Blocks b;
    const double* w = S.z;
    const double* v = S.z + P.ny;
    if (P.heat) {
        const double sk = P.tau * P.qw[l.k];
        b.hy = sk * stencil_sub(P.M, S.y + l.off, S.yd + l.off, l.gx, l.gy);
        b.ktp = op_apply_at(P.Mtl, S.p + l.off, l.gx, l.gy);
        if (l.k + 1 < P.nt) b.ktp -= op_apply_at(P.M, S.p + l.off + P.ns, l.gx, l.gy);
        b.ky = op_apply_at(P.Mtl, S.y + l.off, l.gx, l.gy);
        if (l.k > 0) b.ky -= op_apply_at(P.M, S.y + l.off - P.ns, l.gx, l.gy);
        b.mwv = stencil_sub(P.M, w + l.off, v + l.off, l.gx, l.gy);
        b.mp = op_apply_at(P.M, S.p + l.off, l.gx, l.gy);
        b.hzs = P.alpha * P.tau * P.qw[l.k];
        b.bs = P.tau;
        b.bg = (P.beta * P.tau * P.qw[l.k]) * S.ld[l.i];
    } else {
        b.hy = stencil_sub(P.Mobs, S.y, S.yd, l.gx, l.gy);
        b.ktp = op_apply_at(P.LT, S.p, l.gx, l.gy);
        b.ky = op_apply_at(P.L, S.y, l.gx, l.gy);
        b.mwv = stencil_sub(P.M, w, v, l.gx, l.gy);
        b.mp = op_apply_at(P.M, S.p, l.gx, l.gy);
        b.hzs = P.alpha;
        b.bs = 1.0;
        b.bg = P.beta * S.ld[l.i];
    }
    return b;
}

__global__ void k_theta(ProbDev P, IpmDev S, int* flags)
{
    const long long N = P.ny;
    const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (g < 2 * N) {
        const double lo = S.z[g] - S.za[g];
        const double hi = S.zb[g] - S.z[g];
        if (lo <= 0.0 || hi <= 0.0) atomicOr(flags, kErrThetaZ);
        const double val = S.lza[g] / lo + S.lzb[g] / hi;
        if (g < N) S.tw[g] = val;
        else S.tv[g - N] = val;
    }
    if (P.has_sb && g < N) {
        const double lo = S.y[g] - S.ya[g];
        const double hi = S.yb[g] - S.y[g];
        if (lo <= 0.0 || hi <= 0.0) atomicOr(flags, kErrThetaY);
        S.ty[g] = S.lya[g] / lo + S.lyb[g] / hi;
    }
}

__global__ void k_newton_rhs(ProbDev P, IpmDev S, double mu, double* __restrict__ rhs)
{
    const long long N = P.ny;
    const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= N) return;
    const Loc l = locate(P, g);
    const Blocks b = blocks_at(P, S, l);
    double r1 = b.hy + b.ktp;
    if (P.has_sb) {
        r1 -= mu / (S.y[g] - S.ya[g]);
        r1 += mu / (S.yb[g] - S.y[g]);
    }
    const double hzw = b.hzs * b.mwv;
    const double btp = b.bs * b.mp;
    double r2w = (hzw + b.bg) - btp;
    r2w -= mu / (S.z[g] - S.za[g]);
    r2w += mu / (S.zb[g] - S.z[g]);
    double r2v = (-hzw + b.bg) - (-btp);
    r2v -= mu / (S.z[N + g] - S.za[N + g]);
    r2v += mu / (S.zb[N + g] - S.z[N + g]);
    const double r3 = (b.ky - b.bs * b.mwv) - S.f[g];
    rhs[g] = -r1;
    rhs[N + g] = -r2w;
    rhs[2 * N + g] = -r2v;
    rhs[3 * N + g] = -r3;
}

__device__ __forceinline__ void box_ratio(double x, double dx, double lo, double hi, double& r)
{
    if (dx < 0.0) r = fmin(r, (lo - x) / dx);
    if (dx > 0.0) r = fmin(r, (hi - x) / dx);
}

__device__ __forceinline__ void zero_ratio(double lam, double dlam, double& r)
{
    if (dlam < 0.0) r = fmin(r, -lam / dlam);
}

__global__ void __launch_bounds__(kRedThreads) k_recover_ratios(ProbDev P, IpmDev S, double mu,
                                                                double* __restrict__ part)
{
    __shared__ double sh[32];
    const long long N = P.ny;
    double rp = inf_d(), rd = inf_d();
    for (long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x; g < 2 * N;
         g += (long long)gridDim.x * blockDim.x) {
        const double lo = S.z[g] - S.za[g];
        const double hi = S.zb[g] - S.z[g];
        const double dz = S.dz[g];
        const double la = S.lza[g], lb = S.lzb[g];
        const double dla = -la / lo * dz - la + mu / lo;
        const double dlb = lb / hi * dz - lb + mu / hi;
        S.dlza[g] = dla;
        S.dlzb[g] = dlb;
        box_ratio(S.z[g], dz, S.za[g], S.zb[g], rp);
        zero_ratio(la, dla, rd);
        zero_ratio(lb, dlb, rd);
        if (P.has_sb && g < N) {
            const double ylo = S.y[g] - S.ya[g];
            const double yhi = S.yb[g] - S.y[g];
            const double dy = S.dy[g];
            const double lya = S.lya[g], lyb = S.lyb[g];
            const double dlya = -lya / ylo * dy - lya + mu / ylo;
            const double dlyb = lyb / yhi * dy - lyb + mu / yhi;
            S.dlya[g] = dlya;
            S.dlyb[g] = dlyb;
            box_ratio(S.y[g], dy, S.ya[g], S.yb[g], rp);
            zero_ratio(lya, dlya, rd);
            zero_ratio(lyb, dlyb, rd);
        }
    }
    rp = block_min(rp, sh);
    __syncthreads();
    rd = block_min(rd, sh);
    if (threadIdx.x == 0) {
        part[blockIdx.x] = rp; // block_min leaves the result in thread 0 each time
    }
    // second reduction overwrote sh; recompute rp result stored above is valid
    if (threadIdx.x == 0) part[kRedBlocks + blockIdx.x] = rd;
}

__global__ void k_step_lengths(const double* __restrict__ part, double alpha0, double* steps)
{
    const int lane = threadIdx.x;
    double rp = inf_d(), rd = inf_d();
    for (int i = lane; i < kRedBlocks; i += 32) {
        rp = fmin(rp, part[i]);
        rd = fmin(rd, part[kRedBlocks + i]);
    }
    rp = warp_min(rp);
    rd = warp_min(rd);
    if (lane == 0) {
        steps[0] = fmin(1.0, alpha0 * rp);
        steps[1] = fmin(1.0, alpha0 * rd);
        steps[2] = rp;
        steps[3] = rd;
    }
}

__global__ void k_ipm_update(ProbDev P, IpmDev S, const double* __restrict__ steps, int* flags)
{
    const long long N = P.ny;
    const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const double ap = steps[0], ad = steps[1];
    if (g < 2 * N) {
        const double z = S.z[g] + ap * S.dz[g];
        S.z[g] = z;
        const double la = S.lza[g] + ad * S.dlza[g];
        const double lb = S.lzb[g] + ad * S.dlzb[g];
        S.lza[g] = la;
        S.lzb[g] = lb;
        if (!(z > S.za[g] && z < S.zb[g])) atomicOr(flags, kErrZInterior);
        if (!(la > 0.0)) atomicOr(flags, kErrLamZa);
        if (!(lb > 0.0)) atomicOr(flags, kErrLamZb);
    }
    if (g < N) {
        const double y = S.y[g] + ap * S.dy[g];
        S.y[g] = y;
        S.p[g] = S.p[g] + ad * S.dp[g];
        if (P.has_sb) {
            const double la = S.lya[g] + ad * S.dlya[g];
            const double lb = S.lyb[g] + ad * S.dlyb[g];
            S.lya[g] = la;
            S.lyb[g] = lb;
            if (!(y > S.ya[g] && y < S.yb[g])) atomicOr(flags, kErrYInterior);
            if (!(la > 0.0)) atomicOr(flags, kErrLamYa);
            if (!(lb > 0.0)) atomicOr(flags, kErrLamYb);
        }
    }
}

__global__ void __launch_bounds__(kRedThreads) k_ipm_residuals(ProbDev P, IpmDev S, double mu,
                                                               double* __restrict__ part)
{
    __shared__ double sh[32];
    const long long N = P.ny;
    double sp = 0.0, sd = 0.0, sc = 0.0;
    for (long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x; g < N;
         g += (long long)gridDim.x * blockDim.x) {
        const Loc l = locate(P, g);
        const Blocks b = blocks_at(P, S, l);
        const double xp = (b.ky - b.bs * b.mwv) - S.f[g];
        double xdy = b.hy + b.ktp;
        if (P.has_sb) xdy = (xdy - S.lya[g]) + S.lyb[g];
        const double hzw = b.hzs * b.mwv;
        const double btp = b.bs * b.mp;
        const double xdw = (((hzw + b.bg) - btp) - S.lza[g]) + S.lzb[g];
        const double xdv = (((-hzw + b.bg) - (-btp)) - S.lza[N + g]) + S.lzb[N + g];
        sp += xp * xp;
        sd += xdy * xdy + xdw * xdw + xdv * xdv;
        if (P.has_sb) {
            const double c1 = (S.y[g] - S.ya[g]) * S.lya[g] - mu;
            const double c2 = (S.yb[g] - S.y[g]) * S.lyb[g] - mu;
            sc += c1 * c1 + c2 * c2;
        }
        for (int h = 0; h < 2; ++h) {
            const long long q = g + h * N;
            const double c3 = (S.z[q] - S.za[q]) * S.lza[q] - mu;
            const double c4 = (S.zb[q] - S.z[q]) * S.lzb[q] - mu;
            sc += c3 * c3 + c4 * c4;
        }
    }
    sp = block_sum(sp, sh);
    __syncthreads();
    if (threadIdx.x == 0) part[blockIdx.x] = sp;
    sd = block_sum(sd, sh);
    __syncthreads();
    if (threadIdx.x == 0) part[kRedBlocks + blockIdx.x] = sd;
    sc = block_sum(sc, sh);
    if (threadIdx.x == 0) part[2 * kRedBlocks + blockIdx.x] = sc;
}

__global__ void k_residual_norms(const double* __restrict__ part, double ny, int has_sb,
                                 double* norms)
{
    const double sp = sum_partials_warp(part, kRedBlocks);
    const double sd = sum_partials_warp(part + kRedBlocks, kRedBlocks);
    const double sc = sum_partials_warp(part + 2 * kRedBlocks, kRedBlocks);
    if (threadIdx.x == 0) {
        norms[0] = sqrt(sp) / sqrt(ny);
        norms[1] = sqrt(sd) / sqrt(3.0 * ny);
        norms[2] = sqrt(sc) / sqrt((has_sb ? 2.0 * ny : 0.0) + 4.0 * ny);
    }
}

__global__ void __launch_bounds__(kRedThreads) k_objective(ProbDev P, IpmDev S,
                                                           double* __restrict__ part)
{
    __shared__ double sh[32];
    const long long N = P.ny;
    double a = 0.0, bq = 0.0, c = 0.0, cnt = 0.0, l1 = 0.0;
    const double* w = S.z;
    const double* v = S.z + N;
    for (long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x; g < N;
         g += (long long)gridDim.x * blockDim.x) {
        const Loc l = locate(P, g);
        const double diff = S.y[g] - S.yd[g];
        double hy, m, bg;
        if (P.heat) {
            hy = (P.tau * P.qw[l.k]) * stencil_sub(P.M, S.y + l.off, S.yd + l.off, l.gx, l.gy);
            const double ak = P.alpha * P.tau * P.qw[l.k];
            m = ak * stencil_sub(P.M, w + l.off, v + l.off, l.gx, l.gy);
            bg = (P.beta * P.tau * P.qw[l.k]) * S.ld[l.i];
        } else {
            hy = stencil_sub(P.Mobs, S.y, S.yd, l.gx, l.gy);
            m = stencil_sub(P.M, w, v, l.gx, l.gy);
            bg = P.beta * S.ld[l.i];
        }
        a += diff * hy;
        bq += w[g] * m + v[g] * (-m);
        c += bg * (w[g] + v[g]);
        const double u = w[g] - v[g];
        if (fabs(u) < 1e-2) cnt += 1.0;
        l1 += fabs(u);
    }
    double vals[5] = {a, bq, c, cnt, l1};
    for (int q = 0; q < 5; ++q) {
        const double r = block_sum(vals[q], sh);
        __syncthreads();
        if (threadIdx.x == 0) part[q * kRedBlocks + blockIdx.x] = r;
    }
}

__global__ void k_objective_final(const double* __restrict__ part, int heat, double alpha,
                                  double* out)
{
    double r[5];
    for (int q = 0; q < 5; ++q) r[q] = sum_partials_warp(part + q * kRedBlocks, kRedBlocks);
    if (threadIdx.x == 0) {
        double val = 0.5 * r[0];
        val += heat ? 0.5 * r[1] : 0.5 * alpha * r[1];
        val += r[2];
        out[0] = val;
        out[1] = r[3];
        out[2] = r[4];
    }
}

__global__ void k_initial_point(ProbDev P, IpmDev S)
{
    const long long N = P.ny;
    const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (g < 2 * N) {
        S.z[g] = 0.5 * (S.za[g] + S.zb[g]);
        S.lza[g] = 1.0;
        S.lzb[g] = 1.0;
    }
    if (g < N) {
        double y = S.yd[g];
        if (P.has_sb) {
            const double delta = 1e-2 * (S.yb[g] - S.ya[g]);
            y = fmin(fmax(y, S.ya[g] + delta), S.yb[g] - delta);
            S.lya[g] = 1.0;
            S.lyb[g] = 1.0;
        }
        S.y[g] = y;
        S.p[g] = 0.0;
    }
}

__global__ void k_recover_control(long long N, const double* __restrict__ z, double* __restrict__ u)
{
    const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (g < N) u[g] = z[g] - z[N + g];
}

} // namespace

void launch_theta(cudaStream_t s, const ProbDev& P, const IpmDev& S, int* flags)
{
    note_launch();
    k_theta<<<blocks_for(2 * P.ny), kT, 0, s>>>(P, S, flags);
}

void launch_newton_rhs(cudaStream_t s, const ProbDev& P, const IpmDev& S, double mu, double* rhs)
{
    note_launch();
    k_newton_rhs<<<blocks_for(P.ny), kT, 0, s>>>(P, S, mu, rhs);
}

void launch_recover_ratios(cudaStream_t s, const ProbDev& P, const IpmDev& S, double mu,
                           double* part)
{
    note_launch();
    k_recover_ratios<<<kRedBlocks, kRedThreads, 0, s>>>(P, S, mu, part);
}

void launch_step_lengths(cudaStream_t s, const double* part, double alpha0, double* steps)
{
    note_launch();
    k_step_lengths<<<1, 32, 0, s>>>(part, alpha0, steps);
}

void launch_ipm_update(cudaStream_t s, const ProbDev& P, const IpmDev& S, const double* steps,
                       int* flags)
{
    note_launch();
    k_ipm_update<<<blocks_for(2 * P.ny), kT, 0, s>>>(P, S, steps, flags);
}

void launch_ipm_residuals(cudaStream_t s, const ProbDev& P, const IpmDev& S, double mu,
                          double* part, double* norms)
{
    note_launch();
    k_ipm_residuals<<<kRedBlocks, kRedThreads, 0, s>>>(P, S, mu, part);
    note_launch();
    k_residual_norms<<<1, 32, 0, s>>>(part, (double)P.ny, P.has_sb, norms);
}

void launch_objective(cudaStream_t s, const ProbDev& P, const IpmDev& S, double* part, double* out)
{
    note_launch();
    k_objective<<<kRedBlocks, kRedThreads, 0, s>>>(P, S, part);
    note_launch();
    k_objective_final<<<1, 32, 0, s>>>(part, P.heat, P.alpha, out);
}

// ---------------------------------------------------------- problem setup
// split_bounds (qp.cpp:31-44) with the pinned-bound inflation (qp.cpp:162-166)
// and the bound checks of ControlProblem::validate (qp.cpp:10-28), replicated
// over the time blocks: za = [max(u_a,0); -min(u_b,0)], zb = [max(u_b,0); -min(u_a,0)].
__global__ void k_split_bounds(long long ns, int nt, const double* __restrict__ ua,
                               const double* __restrict__ ub, double* __restrict__ za,
                               double* __restrict__ zb, int* flags)
{
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= ns) return;
    const double a = ua[i], b = ub[i];
    if (a > 0.0 || b < 0.0) atomicOr(flags, kErrCtrlBounds);
    double z[4] = {fmax(a, 0.0), -fmin(b, 0.0), fmax(b, 0.0), -fmin(a, 0.0)};
    for (int h = 0; h < 2; ++h)
        if (z[2 + h] - z[h] < 1e-12) z[2 + h] = z[h] + 1e-12;
    const long long ny = ns * nt;
    for (int k = 0; k < nt; ++k) {
        const long long g = (long long)k * ns + i;
        za[g] = z[0];
        za[ny + g] = z[1];
        zb[g] = z[2];
        zb[ny + g] = z[3];
    }
}

// state box check (y_a <= 0 <= y_b) of ControlProblem::validate
__global__ void k_check_state_bounds(long long n, const double* __restrict__ ya,
                                     const double* __restrict__ yb, int* flags)
{
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n && (ya[i] > 0.0 || yb[i] < 0.0)) atomicOr(flags, kErrStateBounds);
}

// row sums of the eliminated mass from its constant stencil (lumped_diag)
__global__ void k_lumped(int nx, Op9 M, double* __restrict__ ld)
{
    const long long n = (long long)nx * nx;
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int gy = (int)i / nx, gx = (int)i - gy * nx;
    double s = 0.0;
    for (int d = 0; d < 9; ++d) {
        const int jx = gx + d % 3 - 1, jy = gy + d / 3 - 1;
        if (jx < 0 || jx >= nx || jy < 0 || jy >= nx) continue;
        s += M.c[d];
    }
    ld[i] = s;
}

// out[k ns + i] = scale * in[i] for every time block (or a plain copy per block)
__global__ void k_replicate(long long ns, int nt, double scale, const double* __restrict__ in,
                            double* __restrict__ out)
{
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= ns) return;
    const double v = scale * in[i];
    for (int k = 0; k < nt; ++k) out[(long long)k * ns + i] = v;
}

void launch_split_bounds(cudaStream_t s, long long ns, int nt, const double* ua, const double* ub,
                         double* za, double* zb, int* flags)
{
    note_launch();
    k_split_bounds<<<blocks_for(ns), kT, 0, s>>>(ns, nt, ua, ub, za, zb, flags);
}

void launch_check_state_bounds(cudaStream_t s, long long n, const double* ya, const double* yb,
                               int* flags)
{
    note_launch();
    k_check_state_bounds<<<blocks_for(n), kT, 0, s>>>(n, ya, yb, flags);
}

void launch_lumped(cudaStream_t s, int nx, const Op9& M, double* ld)
{
    note_launch();
    k_lumped<<<blocks_for((long long)nx * nx), kT, 0, s>>>(nx, M, ld);
}

void launch_replicate(cudaStream_t s, long long ns, int nt, double scale, const double* in,
                      double* out)
{
    note_launch();
    k_replicate<<<blocks_for(ns), kT, 0, s>>>(ns, nt, scale, in, out);
}

void launch_initial_point(cudaStream_t s, const ProbDev& P, const IpmDev& S)
{
    note_launch();
    k_initial_point<<<blocks_for(2 * P.ny), kT, 0, s>>>(P, S);
}

void launch_recover_control(cudaStream_t s, long long ny, const double* z, double* u)
{
    note_launch();
    k_recover_control<<<blocks_for(ny), kT, 0, s>>>(ny, z, u);
}

} // namespace ocb
