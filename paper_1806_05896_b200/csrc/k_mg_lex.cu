// Lexicographic Gauss-Seidel sweep for the multi-CTA levels (>= 7), the
// reference's own smoother (gauss_seidel_sweep, multigrid.cpp:44-66), run as
// the skewed wavefront described in lex_gs.cuh: one warp per CTA owns 32
// consecutive rows; warp w+1 consumes the last row of warp w through a
// global per-column mailbox (sentinel protocol), prefetched kLexD columns
// ahead so the inter-warp hand-off latency overlaps the sweep.
//
// In place, like the reference. Old values (E and the row above) are read
// through L1: no CTA reads a location another CTA writes in the same sweep,
// except the mailbox, which is accessed with .relaxed.gpu (L2) operations.
#include "kernels.hpp"
#include "lex_gs.cuh"

#include <cstring>

namespace ocb {

namespace {

constexpr int kLexD = 8; // mailbox prefetch distance (columns)

__device__ __forceinline__ double ld_relaxed(const double* p)
{
    double v;
    asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed(double* p, double v)
{
    asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}

template <bool VAR>
__global__ void __launch_bounds__(32) k_gs_lex(Op9 A, const double* __restrict__ b,
                                               const double* __restrict__ inv, double* x, int fwd,
                                               double* mbox, int* flags)
{
    const int nx = A.nx;
    const long long n = (long long)nx * nx;
    const int w = blockIdx.x, j = threadIdx.x;
    const int r = 32 * w + j; // logical row
    const bool rowok = r < nx, hasN = r + 1 < nx;
    const long long sx = fwd ? 1 : -1;                       // physical step of logical x+1
    const long long sy = fwd ? (long long)nx : -(long long)nx; // physical step of logical row+1
    const long long row0 = fwd ? (long long)r * nx : (long long)(nx - 1 - r) * nx + (nx - 1);
    double c[9];
#pragma unroll
    for (int d = 0; d < 9; ++d) c[d] = VAR ? 0.0 : A.c[fwd ? d : 8 - d];
    const bool consumer = j == 0 && w > 0;
    const bool producer = j == 31 && hasN;
    double* mb_in = mbox + (long long)(w > 0 ? w - 1 : 0) * nx;
    double* mb_out = mbox + (long long)w * nx;

    // mailbox ring (lane 0): slot u holds the column congruent to u mod kLexD
    double pf[kLexD];
#pragma unroll
    for (int u = 0; u < kLexD; ++u) pf[u] = (consumer && u < nx) ? ld_relaxed(mb_in + u) : 0.0;

    double sw = 0.0, s = 0.0, se = 0.0; // new row r-1 at x-1, x, x+1
    double last = 0.0;                  // value produced by this lane in the previous step
    double n_prev = 0.0;                // old row r+1 at x-1 (previous step's N)
    int stall = 0;
    const int nsteps = nx + 2 * 31;
    // step st = -1 primes lane 0's window with column 0 of row r-1
    for (int base = -1; base < nsteps; base += kLexD) {
#pragma unroll
        for (int u = 0; u < kLexD; ++u) {
            const int st = base + u;
            const int xl = st - 2 * j;
            double up = __shfl_up_sync(0xffffffffu, last, 1);
            if (j == 0) {
                up = 0.0;
                const int xe = st + 1; // column of row r-1 needed as SE
                if (consumer && xe < nx) {
                    double v = pf[u]; // (base + 1 + u) % kLexD == u
                    while (lex_is_sentinel(v)) {
                        v = ld_relaxed(mb_in + xe);
                        if (++stall > kLexSpinLimit) {
                            atomicOr(flags, kErrLexStall);
                            v = 0.0;
                            break;
                        }
                    }
                    up = v;
                    st_relaxed(mb_in + xe, lex_sentinel());
                    pf[u] = (xe + kLexD < nx) ? ld_relaxed(mb_in + xe + kLexD) : 0.0;
                }
            }
            sw = s;
            s = se;
            se = up;
            double v = 0.0, nn = 0.0;
            if (rowok && xl >= 0 && xl < nx) {
                const long long i = row0 + xl * sx;
                const bool hasE = xl + 1 < nx;
                const double e = hasE ? x[i + sx] : 0.0;
                double ne = 0.0;
                if (hasN) {
                    nn = x[i + sy];
                    if (hasE) ne = x[i + sy + sx];
                }
                auto a = [&](int d) -> double {
                    return VAR ? __ldg(A.coef + (long long)(fwd ? d : 8 - d) * n + i) : c[d];
                };
                v = lex_update(a, __ldg(b + i), __ldg(inv + i), sw, s, se, last, e, n_prev, nn, ne);
                x[i] = v;
                if (producer) st_relaxed(mb_out + xl, v);
            }
            n_prev = nn;
            last = v;
        }
    }
}

} // namespace

void launch_gs_lex(cudaStream_t s, const Op9& A, const double* b, const double* inv, double* x,
                   bool forward, double* mbox, int* flags)
{
    const unsigned nw = (unsigned)((A.nx + 31) / 32);
    note_launch();
    if (A.coef) k_gs_lex<true><<<nw, 32, 0, s>>>(A, b, inv, x, forward ? 1 : 0, mbox, flags);
    else k_gs_lex<false><<<nw, 32, 0, s>>>(A, b, inv, x, forward ? 1 : 0, mbox, flags);
}

double lex_sentinel_host()
{
    double v;
    static_assert(sizeof(v) == sizeof(kLexSentinel), "64-bit sentinel");
    memcpy(&v, &kLexSentinel, sizeof(v));
    return v;
}

} // namespace ocb
