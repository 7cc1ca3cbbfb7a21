// Microbenchmark (tuning aid): one CTA-0 colour pass of the cluster kernel
// (padded planar layout, compile-time neighbour offsets), 256 threads, level
// NX = 31 / 15 / 7, timed over many passes with clock64.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_c0pass tools/ubench_c0pass.cu
#include <cstdio>
#include <cuda_runtime.h>

__host__ __device__ constexpr int fl2(int v) { return (v - (((v % 2) + 2) % 2)) / 2; }
template <int NX>
struct FullG {
    static constexpr int WX = (NX + 1) / 2, SX = WX + 1, PS = (WX + 1) * SX, S = 4 * PS;
    __host__ __device__ static constexpr int xi(int gx, int gy)
    {
        return ((gx & 1) + 2 * (gy & 1)) * PS + (fl2(gy) + 1) * SX + fl2(gx) + 1;
    }
    __host__ __device__ static constexpr int nb(int c, int dx, int dy) { return xi((c & 1) + dx, (c >> 1) + dy); }
};

template <int NX, bool BAR>
__global__ void k(double* out, long long* cyc, int reps)
{
    using G = FullG<NX>;
    extern __shared__ double sm[];
    double* coef = sm;
    double* x = coef + 9 * G::S;
    double* b = x + G::S;
    double* inv = b + G::S;
    for (int i = threadIdx.x; i < 12 * G::S; i += blockDim.x) sm[i] = 0.001 * (i % 97);
    __syncthreads();
    const int t = threadIdx.x;
    const int rr = t / G::WX, cc = t - rr * G::WX;
    const int q = rr * G::SX + cc;
    const bool thr = t < G::WX * G::WX;
    long long t0 = clock64();
    for (int it = 0; it < reps; ++it) {
#pragma unroll
        for (int p = 0; p < 4; ++p) {
            const int c = p;
            const int gx = 2 * cc + (c & 1), gy = 2 * rr + (c >> 1);
            if (thr && gx < NX && gy < NX) {
                const int me = q + G::nb(c, 0, 0);
                double s = b[me];
#pragma unroll
                for (int d = 0; d < 9; ++d) {
                    if (d == 4) continue;
                    s -= coef[d * G::S + me] * x[q + G::nb(c, d % 3 - 1, d / 3 - 1)];
                }
                x[me] = s * inv[me];
            }
            if (BAR) __syncthreads();
            else __syncwarp();
        }
    }
    long long t1 = clock64();
    if (t == 0) cyc[0] = t1 - t0;
    out[t] = x[t];
}

template <int NX, bool BAR>
void run(double* out, long long* cyc, const char* name)
{
    using G = FullG<NX>;
    const int smem = 12 * G::S * 8;
    cudaFuncSetAttribute(k<NX, BAR>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int reps = 2000;
    for (int r = 0; r < 2; ++r) {
        k<NX, BAR><<<1, 256, smem>>>(out, cyc, reps);
        cudaDeviceSynchronize();
    }
    printf("%-28s %.1f cyc/pass\n", name, (double)cyc[0] / (4.0 * reps));
}

int main()
{
    double* out;
    long long* cyc;
    cudaMalloc(&out, 4096 * sizeof(double));
    cudaMallocManaged(&cyc, sizeof(long long));
    run<31, true>(out, cyc, "level 5 (31), bar");
    run<15, true>(out, cyc, "level 4 (15), bar");
    run<7, true>(out, cyc, "level 3 (7), bar");
    run<7, false>(out, cyc, "level 3 (7), syncwarp");
    return 0;
}
