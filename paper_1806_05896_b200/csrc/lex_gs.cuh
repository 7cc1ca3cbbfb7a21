// Lexicographic Gauss-Seidel (the reference smoother, multigrid.cpp:44-66) as
// a skewed wavefront, shared by the multi-CTA sweep kernel (k_mg_lex.cu) and
// the single-CTA bottom solver (k_mg.cu).
//
// Row-major order with x fastest: node (x, y) needs the NEW values of W
// (x-1, y) and SW, S, SE (x-1..x+1, y-1) and the OLD values of E, NW, N, NE.
// Lane j of wavefront warp w owns logical row r = 32 w + j and at step s
// updates logical column x = s - 2 j, so lane j-1 produced (x+1, r-1) one step
// earlier: it arrives by one shuffle per step, and the window of the last
// three shuffled values supplies SW, S, SE. Lane 0 receives row r-1 from the
// previous warp through a per-column mailbox whose slots hold a signalling-NaN
// sentinel until the producer stores the value (the value is its own flag:
// no fences, no cache invalidation); the consumer restores the sentinel after
// reading. Backward sweeps (rows and columns descending) run the same code in
// mirrored coordinates: logical (x, r) is physical (nx-1-x, nx-1-r) and
// stencil entry d becomes 8-d.
//
// Summation order: old-value terms, then SW, S, SE, W, times 1/a_ii. This is
// a reassociation of the reference's loop (rounding-level difference only).
#pragma once

#include "oc_common.cuh"

#include <cstdint>

namespace ocb {

constexpr unsigned long long kLexSentinel = 0x7FF4DEADBEEF5A5Aull; // sNaN: never produced by arithmetic
constexpr int kLexSpinLimit = 1 << 26;                           // polls before declaring a fault

__device__ __forceinline__ bool lex_is_sentinel(double v)
{
    return (unsigned long long)__double_as_longlong(v) == kLexSentinel;
}

__device__ __forceinline__ double lex_sentinel() { return __longlong_as_double((long long)kLexSentinel); }

// x_new = (b - sum_{d != 4} a_d x_d) / a_ii with the old-value terms first.
// a(d) returns the coefficient of LOGICAL stencil entry d.
template <class Coef>
__device__ __forceinline__ double lex_update(const Coef& a, double bval, double inv, double sw,
                                             double s, double se, double w, double e, double nw,
                                             double n, double ne)
{
    double t = bval;
    t -= a(5) * e;
    t -= a(6) * nw;
    t -= a(7) * n;
    t -= a(8) * ne;
    t -= a(0) * sw;
    t -= a(1) * s;
    t -= a(2) * se;
    t -= a(3) * w;
    return t * inv;
}

} // namespace ocb
