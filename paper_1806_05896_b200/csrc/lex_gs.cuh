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
// Arithmetic (lex_update_ref): the reference's gauss_seidel_sweep update
// (multigrid.cpp:49-60) term by term: s = b; s -= a_ij x_j over the row's
// columns in ascending physical order with separate multiply and subtract
// (multigrid.cpp is compiled without FMA contraction); x_i = s / a_ii
// correctly rounded.
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

// s / d correctly rounded from inv = RN(1/d): one Markstein correction with
// the exact FMA remainder (tested equal to div.rn.f64, tests/test_gpu_lex.py).
__device__ __forceinline__ double lex_div_rn(double s, double d, double inv)
{
    const double q0 = __dmul_rn(s, inv);
    const double r = __fma_rn(-q0, d, s);
    return __fma_rn(r, inv, q0);
}

// The reference's node update in logical coordinates: a[0..7] are the
// LOGICAL entries SW,S,SE,W,E,NW,N,NE; forward sweeps subtract them in that
// order, backward (mirrored) sweeps in the reverse order (= physical
// ascending columns).
__device__ __forceinline__ double lex_update_ref(const double* a, bool fwd, double b, double sw,
                                                 double s, double se, double w, double e,
                                                 double nw, double n, double ne, double d,
                                                 double inv)
{
    double t = b;
    if (fwd) {
        t = __dsub_rn(t, __dmul_rn(a[0], sw));
        t = __dsub_rn(t, __dmul_rn(a[1], s));
        t = __dsub_rn(t, __dmul_rn(a[2], se));
        t = __dsub_rn(t, __dmul_rn(a[3], w));
        t = __dsub_rn(t, __dmul_rn(a[4], e));
        t = __dsub_rn(t, __dmul_rn(a[5], nw));
        t = __dsub_rn(t, __dmul_rn(a[6], n));
        t = __dsub_rn(t, __dmul_rn(a[7], ne));
    } else {
        t = __dsub_rn(t, __dmul_rn(a[7], ne));
        t = __dsub_rn(t, __dmul_rn(a[6], n));
        t = __dsub_rn(t, __dmul_rn(a[5], nw));
        t = __dsub_rn(t, __dmul_rn(a[4], e));
        t = __dsub_rn(t, __dmul_rn(a[3], w));
        t = __dsub_rn(t, __dmul_rn(a[2], se));
        t = __dsub_rn(t, __dmul_rn(a[1], s));
        t = __dsub_rn(t, __dmul_rn(a[0], sw));
    }
    return lex_div_rn(t, d, inv);
}

} // namespace ocb
