// Shared device-side definitions for the optcon-b200 kernels (sm_100a, FP64).
//
// Data layout: every field is a dense FP64 vector over the
// interior nodes of a uniform grid, lexicographic with x fastest
// (reference grid.hpp:14-37); time-dependent fields stack nt such blocks
// time-major (timedep.cpp:25-33). Saddle vectors are [y | w | v | p]
// contiguous (ipm.cpp:244-266, precond.cpp:177-198).
#pragma once

#include <cuda_runtime.h>
#include <cstdint>

namespace ocb {

// 9-point operator on one grid level. Entry d = (dy+1)*3 + (dx+1), i.e.
// SW,S,SE,W,C,E,NW,N,NE, which is the ascending CSR column order of a
// lexicographic row in the reference (sparse.hpp:23-74). Neighbours outside
// the interior are Dirichlet-eliminated (fem.cpp:113-140) and contribute 0.
struct Op9 {
    int nx;               // interior nodes per side at this level
    const double* coef;   // 9*n structure-of-arrays coefficients, or nullptr
    double c[9];          // constant stencil (when coef == nullptr)
    const double* diag;   // optional added diagonal (plus_diagonal), or nullptr
    double cscale;        // constant stencil multiplier (1 unless stated)
    const double* csplit; // optional colour-split copy read by the tiled sweep: node
                          // records of 10 words (SW,S,SE,W,E,NW,N,NE, 1/a_ii, pad),
                          // row y holding its even-x nodes first, then its odd-x nodes
};

constexpr int kRedBlocks = 296;   // fixed reduction grid: 2 x 148 SMs (deterministic)
constexpr int kMgsBlocks = 4 * kRedBlocks; // fixed grid of the GMRES orthogonalisation partials
constexpr int kNormBlocks = 2048;           // max grid of the fused multigrid norm checks
constexpr int kRedThreads = 256;

__device__ __forceinline__ double op_coef(const Op9& A, int d, long long i, long long n)
{
    return A.coef ? A.coef[d * n + i] : A.c[d];
}

// (A x)_i with the reference's row summation order (csr_spmv, kernels.cpp:33-45).
// x points at the level's field; gx, gy are 0-based interior coordinates.
// Neighbours outside the interior read as 0 through predicated loads (no
// divergent branches): fma(a, 0, s) == s, so the sum equals skipping them.
__device__ __forceinline__ double op_apply_at(const Op9& A, const double* __restrict__ x, int gx,
                                              int gy)
{
    const int nx = A.nx;
    const int n = nx * nx; // < 2^31 at every level
    const int i = gy * nx + gx;
    const bool hw = gx > 0, he = gx < nx - 1, hs = gy > 0, hn = gy < nx - 1;
    double v[9];
    v[0] = (hs && hw) ? x[i - nx - 1] : 0.0;
    v[1] = hs ? x[i - nx] : 0.0;
    v[2] = (hs && he) ? x[i - nx + 1] : 0.0;
    v[3] = hw ? x[i - 1] : 0.0;
    v[4] = x[i];
    v[5] = he ? x[i + 1] : 0.0;
    v[6] = (hn && hw) ? x[i + nx - 1] : 0.0;
    v[7] = hn ? x[i + nx] : 0.0;
    v[8] = (hn && he) ? x[i + nx + 1] : 0.0;
    double s = 0.0;
    if (A.coef) {
#pragma unroll
        for (int d = 0; d < 9; ++d) {
            double a = A.coef[d * n + i];
            if (d == 4 && A.diag) a += A.diag[i];
            s += a * v[d];
        }
    } else {
#pragma unroll
        for (int d = 0; d < 9; ++d) {
            double a = A.c[d];
            if (d == 4 && A.diag) a += A.diag[i];
            s += a * v[d];
        }
    }
    return s;
}

// Warp/block reductions. All sums use a fixed tree so reruns are
// bit-identical (reference determinism contract, kernels.hpp:20-21).
__device__ __forceinline__ double warp_sum(double v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ double warp_min(double v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_down_sync(0xffffffffu, v, o));
    return v;
}

// Block sum over blockDim.x threads (multiple of 32, <= 1024); result valid in
// thread 0. `sh` must hold 32 doubles.
__device__ __forceinline__ double block_sum(double v, double* sh)
{
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) sh[wid] = v;
    __syncthreads();
    const int nw = blockDim.x >> 5;
    v = (threadIdx.x < nw) ? sh[threadIdx.x] : 0.0;
    if (wid == 0) v = warp_sum(v);
    return v;
}

__device__ __forceinline__ double block_min(double v, double* sh)
{
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    v = warp_min(v);
    __syncthreads();
    if (lane == 0) sh[wid] = v;
    __syncthreads();
    const int nw = blockDim.x >> 5;
    v = (threadIdx.x < nw) ? sh[threadIdx.x] : __longlong_as_double(0x7ff0000000000000LL);
    if (wid == 0) v = warp_min(v);
    return v;
}

// Sum of kRedBlocks partials in a fixed order; every caller gets the same bits.
__device__ __forceinline__ double sum_partials_warp(const double* __restrict__ part, int count)
{
    const int lane = threadIdx.x & 31;
    double v = 0.0;
    for (int i = lane; i < count; i += 32) v += part[i];
    return warp_sum(v); // lane 0 holds the result
}

// Error flags raised on the device and turned into the reference's exception
// types by the host facade (SURVEY.md §5 failure detection).
enum ErrFlag : int {
    kErrMgDiverged = 1 << 0,      // multigrid.cpp:150-154 -> runtime_error
    kErrZInterior = 1 << 1,       // ipm.cpp:313-319 / build_theta -> runtime_error
    kErrYInterior = 1 << 2,
    kErrLamPositive = 1 << 3,
    kErrSingular2x2 = 1 << 4,     // precond.cpp:47-49 -> runtime_error
    kErrNegBracket = 1 << 5,      // precond.cpp:68 -> runtime_error
    kErrBadInput = 1 << 6,        // invalid_argument-class checks on device data
    kErrNonFinite = 1 << 7,
    kErrLamYa = 1 << 8,           // check_positive (ipm.cpp:23-28)
    kErrLamYb = 1 << 9,
    kErrLamZa = 1 << 10,
    kErrLamZb = 1 << 11,
    kErrThetaZ = 1 << 12,         // build_theta (ipm.cpp:44,56)
    kErrThetaY = 1 << 13,
    kErrLexStall = 1 << 14,       // lexicographic wavefront hand-off never arrived
    kErrCtrlBounds = 1 << 15,     // ControlProblem::validate: u_a <= 0 <= u_b
    kErrStateBounds = 1 << 16,    // ControlProblem::validate: y_a <= 0 <= y_b
};

// The block that completes last sums the partials (fixed order) and applies
// the divergence check of MgHierarchy::solve (multigrid.cpp:141-157):
// res = sqrt(sum); flag if res > 10 state[0] (unless init); state[0] = res.
// Every block fences its partial before counting, the last one reads them
// through L2; the counter is reset for the next launch.
__device__ __forceinline__ void finish_norm_check(double* part, unsigned* counter, double* state,
                                                  int* flags, int init)
{
    __shared__ bool last;
    const unsigned nb = gridDim.x * gridDim.y; // partials part[blockIdx.y * gridDim.x + blockIdx.x]
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(counter, 1u) == nb - 1;
    __syncthreads();
    if (!last || threadIdx.x >= 32) return;
    double v = 0.0;
    for (int i = threadIdx.x; i < (int)nb; i += 32) v += __ldcg(part + i);
    v = warp_sum(v);
    if (threadIdx.x == 0) {
        const double res = sqrt(v);
        if (!init && res > 10.0 * state[0]) atomicOr(flags, kErrMgDiverged);
        state[0] = res;
        *counter = 0u;
    }
}

} // namespace ocb
