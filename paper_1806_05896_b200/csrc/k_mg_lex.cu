// Lexicographic Gauss-Seidel sweep for the multi-CTA levels (>= 7), the
// reference's own smoother (gauss_seidel_sweep, multigrid.cpp:44-66), in
// place, with the reference's arithmetic: every node update is
//   s = b_i; s -= a_ij x_j for j in ascending column order; x_i = s / a_ii
// with separate multiply and subtract (the reference's multigrid.cpp is
// compiled without FMA contraction) and a correctly rounded quotient.
//
// Skewed wavefront (lex_gs.cuh): one compute warp per CTA owns 32
// consecutive rows (a band); lane j owns logical row r = 32 w + j and at step
// s updates logical column x = s - 2 j, so lane j-1 produced (x+1, r-1) one
// step earlier and hands it over by one shuffle. Lane 31 writes each new
// value of the band's last row to a global per-column mailbox; band w+1
// fetches it one 16-column chunk ahead (signalling-NaN sentinel protocol:
// the value is its own flag, the consumer restores the sentinels at exit).
//
// Operand staging: the lanes of a step read 32 different rows, so per-lane
// global loads would touch 32 cache lines per instruction. The band is staged
// through shared memory in "parallelogram" chunks instead: chunk c holds, for
// band row rho, the logical columns [16 c - 2 rho, 16 c - 2 rho + 16) of b,
// 1/a_ii, a_ii, the 8 off-diagonal coefficient planes (variable operators)
// and the old x (rows 0..32: row 32 is the next band's first row, the N
// neighbours of lane 31). All lanes consume chunk c during the same 16 steps
// and the row segments are contiguous in global memory (coalesced). Warp
// specialisation: staging warps load each chunk two periods ahead into
// registers (double-buffered), store it into a 4-slot ring, write retired
// chunks back with coalesced stores and fetch the mailbox chunk, while the
// compute warp only runs the 16 dependent steps; one block barrier per chunk.
// New values overwrite the old x in the tile (an old value is dead once its
// own lane moved past it). Nothing another band reads in the same sweep is
// written before it is read: a band lags the band above by >= ~5 chunks
// (it needs the mailbox chunk ahead) and reads the rows of the band below
// (its row 32) at most 4 chunks ahead.
//
// Pipelined batches: the 5 sweeps of a smoothing phase are 5 launches on 5
// streams (Hierarchy::lex_sweeps). Sweep q+1 reads what sweep q wrote, so its
// staging warps wait, before loading chunk c, until sweep q's same band has
// written chunk c back and the band below chunk c-4 (the columns of its first
// row that chunk c stages as row 32); a band publishes its written-back chunk
// count after each period's barrier (fence + relaxed store, acquire loads on
// the other side). Each sweep has its own mailbox set. Sweep q+1 then trails
// sweep q by a few chunks per band instead of a whole sweep (level 10:
// 5 sweeps in ~1.2 sweep times), and nothing it overwrites is still needed by
// sweep q: band w of sweep q+1 writes chunk c only after sweep q's band w wrote
// it, which is after sweep q's band w-1 read it as its row 32. Every wait
// points to an earlier launch or an earlier block of the same launch, so the
// earliest unfinished block can always run (no deadlock when the 160 blocks of
// a level-10 batch exceed the 148 SMs).
//
// Backward sweeps (rows and columns descending) run the same code in
// mirrored coordinates: logical (x, r) is physical (nx-1-x, nx-1-r) and
// stencil entry d becomes 8-d; the physical ascending column order is then
// the logical descending order, which the update follows.
#include "kernels.hpp"
#include "lex_gs.cuh"

#include <atomic>
#include <type_traits>
#include <cstring>

namespace ocb {

namespace {

constexpr int kLW = 16;     // chunk width (columns); all lanes consume a chunk in kLW steps
constexpr int kLP = 17;     // shared row pitch (doubles): lane stride 17 words, conflict-free
constexpr int kLRing = 4;   // chunk slots: current, next (look-ahead), two in flight

// staged per-node arrays: b, 1/a_ii, a_ii, then the 8 off-diagonal planes;
// x has 33 rows. After the ring: the mailbox values of each slot's chunk.
template <bool VAR>
struct LexSlot {
    static constexpr int kArr = VAR ? 11 : 3;
    static constexpr int kDoubles = (kArr * 32 + 33) * kLP;
    static constexpr int kStageWarps = VAR ? 8 : 4; // staging warps next to the compute warp
    static constexpr int kThreads = 32 * (1 + kStageWarps);
    static constexpr size_t kBytes = ((size_t)kLRing * kDoubles + kLRing * kLW + 8) * sizeof(double);
};

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

__device__ __forceinline__ void st_relaxed_if(double* p, double v, bool pred)
{
    asm volatile("{ .reg .pred q; setp.ne.b32 q, %2, 0; @q st.relaxed.gpu.global.f64 [%0], %1; }" ::"l"(p),
                 "d"(v), "r"((int)pred)
                 : "memory");
}
// tuning aid: %globaltimer stamps per band (lane 0): start, after the
// start-up wait, end of chunks 1, 4, 16, end of the main loop
__device__ int g_lex_probe_on = 0;
__device__ unsigned long long g_lex_probe[64 * 8];
__device__ __forceinline__ void lex_stamp(int on, int band, int slot, int tid = 0)
{
    if (on && threadIdx.x == tid && band < 64) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g_lex_probe[band * 8 + slot] = t;
    }
}

struct LexArgs {
    int nx;
    const double* b;
    const double* inv;
    const double* dfull; // a_ii (center coefficient + added diagonal, as the CSR diagonal value)
    const double* coef;  // 9 planes (variable operators) or nullptr
    double c[9];         // constant stencil (physical order)
    double* x;
    double* mbox;
    int* flags;
    int start_col; // column of the band above that starts a band (hand-over lag)
    // Pipelined sweeps (several sweeps of one level in flight, one launch each on
    // its own stream): prog_prev[band] = chunks the PREVIOUS sweep's band has
    // written back (nullptr: nothing to wait for), prog_out[band] = this sweep's.
    const int* prog_prev;
    int* prog_out;
};

__device__ __forceinline__ int ld_acquire_int(const int* p)
{
    int v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
constexpr int kLexDone = 1 << 28; // progress value of a finished band

template <bool VAR, bool FWD>
__global__ void __launch_bounds__(LexSlot<VAR>::kThreads, 1) k_gs_lex(LexArgs a)
{
    extern __shared__ double sm[];
    using Slot = LexSlot<VAR>;
    constexpr int NA = Slot::kArr;
    constexpr int NSW = Slot::kStageWarps;
    const int nx = a.nx;
    const int n = nx * nx; // < 2^31 at every level
    const int w = blockIdx.x;
    const int warp = threadIdx.x >> 5, j = threadIdx.x & 31;
    const int nchunks = (nx + 62 + kLW - 1) / kLW;
    const int probe = g_lex_probe_on;
    double* mbs = sm + kLRing * Slot::kDoubles; // [kLRing][kLW] mailbox values, then column 0
    const bool consumer = w > 0;
    const bool produces = 32 * w + 31 < nx - 1; // band w+1 exists
    const double* mb_in = a.mbox + (size_t)(w > 0 ? w - 1 : 0) * nx;
    double* mb_out = a.mbox + (size_t)w * nx;
    if (warp == 0) lex_stamp(probe, w, 0);

    if (warp > 0) {
        // ================= staging warps: operands in, new values out =====
        // Lane (l, h) of staging warp sw handles column l of band rows
        // rho = 2p + h for row pairs p = sw, sw + NSW, ... (and row 32 of x).
        // The logical position (16c - 2rho + l, 32w + rho) has a physical
        // index affine in p (step di) and c (step dc).
        const int sw = warp - 1;
        const int l = j & 15, h = j >> 4;
        const int rho_lim = nx - 32 * w; // band rows with rho < rho_lim exist
        const int di = FWD ? 2 * nx - 4 : -(2 * nx - 4);
        const int dc = FWD ? kLW : -kLW;
        const int i00 = FWD ? (32 * w + h) * nx + (l - 2 * h)
                            : (nx - 1 - (32 * w + h)) * nx + (nx - 1 - (l - 2 * h));
        const double* planes[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int d = k < 4 ? k : k + 1; // logical entry
            planes[k] = VAR ? a.coef + (size_t)(FWD ? d : 8 - d) * n : a.b;
        }
        // operands of one chunk for this lane, double-buffered in registers:
        // loaded two periods before they are stored to shared memory, so the
        // loads' latency (L2 or DRAM) hides behind two chunks of wavefront
        constexpr int NP = 16 / NSW; // row pairs per staging warp
        double reg[2][NP][NA + 1];
        double reg32[2] = {0.0, 0.0};
        int pstall = 0;
        // previous sweep of a pipelined batch: chunk c of this band reads its own
        // rows after that sweep (its band w wrote chunk c back) and, as row 32,
        // columns [16c - 64, 16c - 48) of band w+1's first row (its chunk c - 4)
        auto wait_prev = [&](int c) {
            if (!a.prog_prev) return;
            if (j == 0) {
                const int need0 = min(c + 1, nchunks), need1 = min(c - 3, nchunks);
                while (ld_acquire_int(a.prog_prev + w) < need0)
                    if (++pstall > kLexSpinLimit) {
                        atomicOr(a.flags, kErrLexStall);
                        break;
                    }
                if (produces && need1 > 0)
                    while (ld_acquire_int(a.prog_prev + w + 1) < need1)
                        if (++pstall > kLexSpinLimit) {
                            atomicOr(a.flags, kErrLexStall);
                            break;
                        }
            }
            __syncwarp();
        };
        auto publish = [&](int done) { // after a barrier that follows the write-backs
            if (a.prog_out && sw == 0 && j == 0) {
                __threadfence();
                asm volatile("st.relaxed.gpu.global.s32 [%0], %1;" ::"l"(a.prog_out + w), "r"(done) : "memory");
            }
        };
        auto load = [&](int c, auto bufc) {
            constexpr int B = decltype(bufc)::value;
            const int ic = i00 + c * dc;
            wait_prev(c);
#pragma unroll
            for (int t = 0; t < NP; ++t) {
                const int p = sw + t * NSW;
                const int rho = 2 * p + h;
                const int xl = kLW * c - 2 * rho + l;
                const bool ok = c <= nchunks && rho < rho_lim && xl >= 0 && xl < nx;
                const int i = ok ? ic + p * di : 0;
                reg[B][t][0] = ok ? __ldcg(a.x + i) : 0.0;
                reg[B][t][1] = ok ? __ldg(a.b + i) : 0.0;
                reg[B][t][2] = ok ? __ldg(a.inv + i) : 0.0;
                reg[B][t][3] = ok ? __ldg(a.dfull + i) : 0.0;
                if (VAR) {
#pragma unroll
                    for (int k = 0; k < 8; ++k)
                        reg[B][t][4 + k] = ok ? __ldg(planes[k] + i) : 0.0;
                }
            }
            if (sw == NSW - 1 && h == 0) { // row 32 of x: the next band's first row
                const int xl = kLW * c - 64 + l;
                const bool ok = c <= nchunks && 32 < rho_lim && xl >= 0 && xl < nx;
                reg32[B] = ok ? __ldcg(a.x + ic + 16 * di) : 0.0;
            }
        };
        auto store = [&](int c, auto bufc) {
            constexpr int B = decltype(bufc)::value;
            double* S = sm + (c % kLRing) * Slot::kDoubles;
            double* X = S + NA * 32 * kLP;
#pragma unroll
            for (int t = 0; t < NP; ++t) {
                const int rho = 2 * (sw + t * NSW) + h;
                double* row = S + rho * kLP + l;
                X[rho * kLP + l] = reg[B][t][0];
                row[0] = reg[B][t][1];
                row[32 * kLP] = reg[B][t][2];
                row[64 * kLP] = reg[B][t][3];
                if (VAR) {
#pragma unroll
                    for (int k = 0; k < 8; ++k) row[(3 + k) * 32 * kLP] = reg[B][t][4 + k];
                }
            }
            if (sw == NSW - 1 && h == 0) X[32 * kLP + l] = reg32[B];
        };
        auto writeback = [&](int c) {
            const double* X = sm + (c % kLRing) * Slot::kDoubles + NA * 32 * kLP;
            const int ic = i00 + c * dc;
#pragma unroll
            for (int p = sw; p < 16; p += NSW) {
                const int rho = 2 * p + h;
                const int xl = kLW * c - 2 * rho + l;
                if (rho < rho_lim && xl >= 0 && xl < nx) a.x[ic + p * di] = X[rho * kLP + l];
            }
        };
        // mailbox values of chunk c (columns 16c + 1 + l) into mbs[c % kLRing]
        int stall = 0;
        auto mailbox = [&](int c) {
            if (!consumer || sw != 0) return;
            const int col = kLW * c + 1 + j;
            double v = 0.0;
            if (j < kLW && col < nx) {
                v = ld_relaxed(mb_in + col);
                while (lex_is_sentinel(v)) {
                    v = ld_relaxed(mb_in + col);
                    if (++stall > kLexSpinLimit) {
                        atomicOr(a.flags, kErrLexStall);
                        v = 0.0;
                    }
                }
            }
            if (j < kLW) mbs[(c % kLRing) * kLW + j] = v;
        };
        using B0 = std::integral_constant<int, 0>;
        using B1 = std::integral_constant<int, 1>;
        load(0, B0{});
        store(0, B0{});
        load(1, B1{});
        store(1, B1{});
        load(2, B0{});
        load(3, B1{});
        if (consumer && sw == 0) {
            // start once the band above has produced column g_lex_start (the
            // lag this sets keeps the next mailbox chunk, fetched at the end
            // of each period, about ready when it is fetched)
            const int xs = min(a.start_col, nx - 1);
            while (lex_is_sentinel(ld_relaxed(mb_in + xs))) {
                if (++stall > kLexSpinLimit) {
                    if (j == 0) atomicOr(a.flags, kErrLexStall);
                    break;
                }
            }
            if (j == 0) { // column 0 (SE of step -1)
                double v0 = ld_relaxed(mb_in);
                while (lex_is_sentinel(v0)) {
                    v0 = ld_relaxed(mb_in);
                    if (++stall > kLexSpinLimit) {
                        atomicOr(a.flags, kErrLexStall);
                        v0 = 0.0;
                    }
                }
                mbs[kLRing * kLW] = v0;
            }
        }
        mailbox(0);
        __syncthreads();
        // period c: write back chunk c-1, store chunk c+2 (loaded in period
        // c-2, buffer c % 2) into the slot chunk c-2 left, load chunk c+4
        // into the same buffer, fetch the mailbox chunk c+1
        auto period = [&](int c, auto bufc) {
            if (c >= 1) writeback(c - 1);
            store(c + 2, bufc);
            load(c + 4, bufc);
            mailbox(c + 1);
            __syncthreads();
            publish(c); // chunks 0 .. c-1 are in global memory
        };
#pragma unroll 1
        for (int c = 0; c < nchunks; c += 2) {
            period(c, B0{});
            if (c + 1 < nchunks) period(c + 1, B1{});
        }
        writeback(nchunks - 1);
        if (a.prog_out) {
            asm volatile("bar.sync 1, %0;" ::"r"(NSW * 32) : "memory"); // the staging warps
            publish(kLexDone);
        }
        // every value of the band above has been consumed (its producer is
        // done): restore the sentinels in one coalesced pass
        if (consumer)
            for (int xq = sw * 32 + j; xq < nx; xq += NSW * 32) const_cast<double*>(mb_in)[xq] = lex_sentinel();
        return;
    }

    // ================= compute warp: the wavefront ====================
    // constant stencil in logical order
    double cst[9];
#pragma unroll
    for (int d = 0; d < 9; ++d) cst[d] = VAR ? 0.0 : a.c[FWD ? d : 8 - d];
    const bool p31 = produces && j == 31; // writes the band's last row to the mailbox
    __syncthreads(); // prologue staged
    lex_stamp(probe, w, 1);

    // registers: new values of row r-1 at x-1, x, x+1; this lane's last value
    // (W); old values of row r+1 at x-1, x (the N window)
    double sw = 0.0, s = 0.0, se = 0.0, last = 0.0;
    if (j == 0 && consumer) se = mbs[kLRing * kLW];
    double nw, nn;
    {
        const double* X0 = sm + NA * 32 * kLP;
        nw = X0[(j + 1) * kLP + 1];
        nn = X0[(j + 1) * kLP + 2];
    }
#pragma unroll 1
    for (int c = 0; c < nchunks; ++c) {
        double* S = sm + (c % kLRing) * Slot::kDoubles;
        double* Sn = sm + ((c + 1) % kLRing) * Slot::kDoubles;
        double* X = S + NA * 32 * kLP;
        double* Xn = Sn + NA * 32 * kLP;
        const double* Sr = S + j * kLP; // this lane's row in the slot's arrays
        const double* mrow = mbs + (c % kLRing) * kLW;
#pragma unroll
        for (int k = 0; k < kLW; ++k) {
            const int xl = kLW * c + k - 2 * j;
            const double bv = Sr[k];
            const double iv = Sr[32 * kLP + k];
            const double dv = Sr[64 * kLP + k];
            double ac[9];
#pragma unroll
            for (int d = 0; d < 9; ++d) {
                const int kk = d < 4 ? d : d - 1;
                ac[d] = (VAR && d != 4) ? Sr[(3 + kk) * 32 * kLP + k] : cst[d];
            }
            const double e = (k + 1 < kLW) ? X[j * kLP + k + 1] : Xn[j * kLP + k + 1 - kLW];
            const double ne = (k + 3 < kLW) ? X[(j + 1) * kLP + k + 3] : Xn[(j + 1) * kLP + k + 3 - kLW];
            const double mv = mrow[k]; // band above, column 16c + k + 1
            // new value of row r-1 at x+1 (SE): lane j-1's last result, or
            // (lane 0) the band above's value from the mailbox chunk
            double up = __shfl_up_sync(0xffffffffu, last, 1);
            up = j == 0 ? (consumer ? mv : 0.0) : up;
            sw = s;
            s = se;
            se = up;
            double t = bv;
            if (FWD) {
                // physical ascending order: SW, S, SE, W, E, NW, N, NE
                t = __dsub_rn(t, __dmul_rn(ac[0], sw));
                t = __dsub_rn(t, __dmul_rn(ac[1], s));
                t = __dsub_rn(t, __dmul_rn(ac[2], se));
                t = __dsub_rn(t, __dmul_rn(ac[3], last));
                t = __dsub_rn(t, __dmul_rn(ac[5], e));
                t = __dsub_rn(t, __dmul_rn(ac[6], nw));
                t = __dsub_rn(t, __dmul_rn(ac[7], nn));
                t = __dsub_rn(t, __dmul_rn(ac[8], ne));
            } else {
                // mirrored: physical ascending = logical NE, N, NW, E, W, SE, S, SW
                t = __dsub_rn(t, __dmul_rn(ac[8], ne));
                t = __dsub_rn(t, __dmul_rn(ac[7], nn));
                t = __dsub_rn(t, __dmul_rn(ac[6], nw));
                t = __dsub_rn(t, __dmul_rn(ac[5], e));
                t = __dsub_rn(t, __dmul_rn(ac[3], last));
                t = __dsub_rn(t, __dmul_rn(ac[2], se));
                t = __dsub_rn(t, __dmul_rn(ac[1], s));
                t = __dsub_rn(t, __dmul_rn(ac[0], sw));
            }
            // branch-free: positions outside the grid were staged as zeros
            // (b, a_ii, 1/a_ii, coefficients), so their quotient is exactly 0
            // (t * 0 = 0, remainder t, fma(t, 0, 0) = 0) and they stay 0
            const double v = lex_div_rn(t, dv, iv);
            X[j * kLP + k] = v;
            // lane 31: the band's last row straight to the band below's mailbox
            const bool put = p31 && xl >= 0 && xl < nx;
            st_relaxed_if(mb_out + (put ? xl : 0), v, put);
            last = v;
            nw = nn;
            nn = ne;
        }
        __syncthreads(); // chunk c done; chunks c+1, c+2 staged
        if (c == 8) lex_stamp(probe, w, 2);
    }
    lex_stamp(probe, w, 5);
}

template <bool VAR, bool FWD>
void go(cudaStream_t s, const LexArgs& a)
{
    constexpr size_t smem = LexSlot<VAR>::kBytes;
    // per device, once (several devices may run in one process)
    static std::atomic<unsigned> done{0};
    int dev = 0;
    cudaGetDevice(&dev);
    const unsigned bit = 1u << (dev & 31);
    if (!(done.load() & bit)) {
        cudaFuncSetAttribute(k_gs_lex<VAR, FWD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        done.fetch_or(bit);
    }
    const unsigned nb = (unsigned)((a.nx + 31) / 32);
    k_gs_lex<VAR, FWD><<<nb, LexSlot<VAR>::kThreads, smem, s>>>(a);
}

} // namespace

std::atomic<int> g_lex_bottom_top{4};
std::atomic<int> g_lex_start{17};
std::atomic<int> g_lex_pipeline{1}; // 1: the sweeps of a smoothing phase run as a pipelined batch

void launch_gs_lex(cudaStream_t s, const Op9& A, const double* b, const double* inv,
                   const double* dfull, double* x, bool forward, double* mbox, int* flags,
                   const int* prog_prev, int* prog_out)
{
    LexArgs a{};
    a.prog_prev = prog_prev;
    a.prog_out = prog_out;
    a.nx = A.nx;
    a.b = b;
    a.inv = inv;
    a.dfull = dfull;
    a.coef = A.coef;
    for (int d = 0; d < 9; ++d) a.c[d] = A.c[d];
    a.x = x;
    a.mbox = mbox;
    a.flags = flags;
    a.start_col = g_lex_start.load();
    note_launch();
    if (A.coef) {
        if (forward) go<true, true>(s, a);
        else go<true, false>(s, a);
    } else {
        if (forward) go<false, true>(s, a);
        else go<false, false>(s, a);
    }
}

void lex_probes(int enable, unsigned long long* out512)
{
    cudaDeviceSynchronize();
    if (out512) cudaMemcpyFromSymbol(out512, g_lex_probe, sizeof(unsigned long long) * 512);
    cudaMemcpyToSymbol(g_lex_probe_on, &enable, sizeof(int));
}

double lex_sentinel_host()
{
    double v;
    static_assert(sizeof(v) == sizeof(kLexSentinel), "64-bit sentinel");
    memcpy(&v, &kLexSentinel, sizeof(v));
    return v;
}

// Test hook: the correctly rounded quotient used by the lexicographic update
// against the IEEE division, elementwise (mismatch count in *bad).
__global__ void k_lex_div_check(const double* s, const double* d, long long n, unsigned long long* bad)
{
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const double inv = 1.0 / d[i];
        const double q = lex_div_rn(s[i], d[i], inv);
        const double ref = __ddiv_rn(s[i], d[i]);
        if (__double_as_longlong(q) != __double_as_longlong(ref)) atomicAdd(bad, 1ull);
    }
}

void launch_lex_div_check(cudaStream_t s, const double* num, const double* den, long long n,
                          unsigned long long* bad)
{
    note_launch();
    k_lex_div_check<<<592, 256, 0, s>>>(num, den, n, bad);
}

} // namespace ocb
