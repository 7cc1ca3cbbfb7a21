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

constexpr int kLexD = 8;    // mailbox prefetch distance (columns)
constexpr int kLexLag = 24; // extra start-up lag of a consumer warp (columns)

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

// Raw operands of a column, loaded kLexD steps before the column is updated
// (the loads never sit on the wavefront's critical path): b, the old values
// E, NW, N, NE, 1/a_ii and, for variable operators, the 8 off-diagonal
// coefficients. Reading them early is exact: the row above (lane j+1) and
// this lane's own row east of the current column are only written later.
// prefetch.L1 runs kLexPF columns ahead so these loads hit L1.
constexpr int kLexPF = 0; // L1 prefetch distance (0: off; uncoalesced prefetches cost L1 bandwidth)

template <bool VAR>
struct LexRaw {
    double b, e, nw, nn, ne, inv;
    double a[VAR ? 8 : 1];
};

__device__ __forceinline__ void prefetch_l1(const void* p)
{
    asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}

template <bool VAR>
__device__ __forceinline__ void lex_load(LexRaw<VAR>& p, const Op9& A, const double* __restrict__ b,
                                         const double* __restrict__ inv, const double* x,
                                         long long n, long long row0, long long sx, long long sy,
                                         int nx, bool rowok, bool hasN, int fwd, int col)
{
    p.b = p.e = p.nw = p.nn = p.ne = p.inv = 0.0;
    if (VAR) {
#pragma unroll
        for (int k = 0; k < (VAR ? 8 : 1); ++k) p.a[k] = 0.0;
    }
    if (!rowok || col < 0 || col >= nx) return;
    const long long i = row0 + col * sx;
    const bool hasE = col + 1 < nx, hasW = col > 0;
    if (kLexPF > 0 && col + kLexPF < nx) {
        const long long ip = i + kLexPF * sx;
        prefetch_l1(b + ip);
        prefetch_l1(inv + ip);
        prefetch_l1(x + ip);
        if (hasN) prefetch_l1(x + ip + sy);
        if (VAR) {
#pragma unroll
            for (int d = 0; d < 9; ++d)
                if (d != 4) prefetch_l1(A.coef + (long long)d * n + ip);
        }
    }
    if (hasE) p.e = x[i + sx];
    if (hasN) {
        p.nn = x[i + sy];
        if (hasW) p.nw = x[i + sy - sx];
        if (hasE) p.ne = x[i + sy + sx];
    }
    p.b = __ldg(b + i);
    p.inv = __ldg(inv + i);
    if (VAR) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int d = k < 4 ? k : k + 1; // logical entry
            p.a[k] = __ldg(A.coef + (long long)(fwd ? d : 8 - d) * n + i);
        }
    }
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
    const long long sx = fwd ? 1 : -1;                         // physical step of logical x+1
    const long long sy = fwd ? (long long)nx : -(long long)nx; // physical step of logical row+1
    const long long row0 = fwd ? (long long)r * nx : (long long)(nx - 1 - r) * nx + (nx - 1);
    double c[9];
#pragma unroll
    for (int d = 0; d < 9; ++d) c[d] = VAR ? 0.0 : A.c[fwd ? d : 8 - d];
    const bool consumer = j == 0 && w > 0;
    const bool producer = j == 31 && hasN;
    double* mb_in = mbox + (long long)(w > 0 ? w - 1 : 0) * nx;
    double* mb_out = mbox + (long long)w * nx;

    int stall = 0;
    // Start kLexLag columns behind the producer: the natural lag (63 steps)
    // would leave the consumer polling L2 for every column; with the extra
    // slack the ring's prefetched mailbox loads already hold produced values.
    if (consumer) {
        const int xs = min(kLexLag, nx - 1);
        while (lex_is_sentinel(ld_relaxed(mb_in + xs))) {
            if (++stall > kLexSpinLimit) {
                atomicOr(flags, kErrLexStall);
                break;
            }
        }
    }
    __syncwarp();
    // mailbox ring (lane 0): slot q holds the column congruent to q mod kLexD
    double pf[kLexD];
#pragma unroll
    for (int q = 0; q < kLexD; ++q) pf[q] = (consumer && q < nx) ? ld_relaxed(mb_in + q) : 0.0;
    // returns row r-1 at column xe (lane 0 of a consumer warp), restoring the sentinel
    auto receive = [&](int q, int xe) -> double {
        double v = pf[q];
        while (lex_is_sentinel(v)) {
            v = ld_relaxed(mb_in + xe);
            if (++stall > kLexSpinLimit) {
                atomicOr(flags, kErrLexStall);
                v = 0.0;
                break;
            }
        }
        st_relaxed(mb_in + xe, lex_sentinel());
        pf[q] = (xe + kLexD < nx) ? ld_relaxed(mb_in + xe + kLexD) : 0.0;
        return v;
    };

    double sw = 0.0, s = 0.0, se = 0.0; // new row r-1 at x-1, x, x+1
    double last = 0.0;                  // this lane's value from the previous step (W)
    // step -1 primes lane 0's window with column 0 of row r-1
    {
        double up = __shfl_up_sync(0xffffffffu, last, 1);
        if (j == 0) up = consumer ? receive(0, 0) : 0.0;
        se = up;
    }
    // operands loaded R steps ahead; ring slot u % R serves steps st = u (mod R)
    constexpr int R = VAR ? 4 : kLexD; // variable operators carry 8 more words per slot
    static_assert(kLexD % R == 0, "ring size divides the unroll");
    LexRaw<VAR> ring[R];
#pragma unroll
    for (int u = 0; u < R; ++u)
        lex_load<VAR>(ring[u], A, b, inv, x, n, row0, sx, sy, nx, rowok, hasN, fwd, u - 2 * j);
    // logical coefficient d of the column in slot q
#define LEX_A(q, d) (VAR ? ring[q].a[(d) < 4 ? (d) : (d) - 1] : c[d])
    const int nsteps = nx + 2 * 31;
    for (int base = 0; base < nsteps; base += kLexD) {
#pragma unroll
        for (int u = 0; u < kLexD; ++u) {
            const int st = base + u;
            const int xl = st - 2 * j;
            const int q = u % R;
            // old-value part first (independent of the wavefront)
            double t = ring[q].b;
            t -= LEX_A(q, 5) * ring[q].e;
            t -= LEX_A(q, 6) * ring[q].nw;
            t -= LEX_A(q, 7) * ring[q].nn;
            t -= LEX_A(q, 8) * ring[q].ne;
            double up = __shfl_up_sync(0xffffffffu, last, 1);
            if (j == 0) {
                const int xe = st + 1; // column of row r-1 needed as SE
                up = (consumer && xe < nx) ? receive((u + 1) % kLexD, xe) : 0.0;
            }
            sw = s;
            s = se;
            se = up;
            double v = 0.0;
            if (rowok && xl >= 0 && xl < nx) {
                t -= LEX_A(q, 0) * sw;
                t -= LEX_A(q, 1) * s;
                t -= LEX_A(q, 2) * se;
                t -= LEX_A(q, 3) * last;
                v = t * ring[q].inv;
                x[row0 + xl * sx] = v;
                if (producer) st_relaxed(mb_out + xl, v);
            }
            last = v;
            lex_load<VAR>(ring[q], A, b, inv, x, n, row0, sx, sy, nx, rowok, hasN, fwd, xl + R);
        }
    }
#undef LEX_A
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
