// Microbenchmark (tuning aid): cost of one Gauss-Seidel colour pass in shared
// memory (LDS of b and 8 neighbours, 8-DFMA chain, STS, __syncthreads), as in
// the cluster kernel's CTA-0 levels, with variants isolating each part.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_pass tools/ubench_pass.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE, int NACT, int ACC = 1>
__global__ void k_pass(double* out, long long* cyc, int passes)
{
    __shared__ double x[4 * 17 * 17];
    __shared__ double cf[9 * 4 * 17 * 4];
    __shared__ double bb[4 * 17 * 17];
    for (int i = threadIdx.x; i < 4 * 17 * 17; i += blockDim.x) { x[i] = 0.001 * i; bb[i] = 1.0; }
    for (int i = threadIdx.x; i < 9 * 4 * 17 * 4; i += blockDim.x) cf[i] = -0.1;
    __syncthreads();
    const int t = threadIdx.x;
    const int q = (t / 16) * 17 + (t % 16);
    long long t0 = clock64();
    for (int p = 0; p < passes; ++p) {
        const int c = p & 3;
        if (MODE != 2 && t < NACT) {
            const int me = c * 289 + 18 + q;
            double s = bb[me], s2 = 0.0;
#pragma unroll
            for (int d = 0; d < 9; ++d) {
                if (d == 4) continue;
                const int off = ((c + d) & 3) * 289 + (d / 3) * 17 + (d % 3);
                if (ACC == 2 && d > 4) s2 += cf[d * 272 + (me & 255)] * x[q + off];
                else s -= cf[d * 272 + (me & 255)] * x[q + off];
            }
            x[me] = (ACC == 2 ? s - s2 : s) * 0.25;
        }
        if (MODE == 3) __syncwarp();
        else if (MODE != 1) __syncthreads();
    }
    long long t1 = clock64();
    if (t == 0) cyc[0] = t1 - t0;
    out[t] = x[t];
}

int main()
{
    double* out;
    long long* cyc;
    cudaMalloc(&out, 4096 * sizeof(double));
    cudaMallocManaged(&cyc, sizeof(long long));
    const int P = 4000;
    auto run = [&](auto kern, const char* name) {
        for (int rep = 0; rep < 2; ++rep) {
            kern<<<1, 256>>>(out, cyc, P);
            cudaDeviceSynchronize();
        }
        printf("%-40s %.1f cyc/pass\n", name, (double)cyc[0] / P);
    };
    run(k_pass<0, 256>, "full pass, 256 active");
    run(k_pass<0, 64>, "full pass, 64 active");
    run(k_pass<0, 16>, "full pass, 16 active");
    run(k_pass<1, 256>, "no barrier, 256 active");
    run(k_pass<1, 16>, "no barrier, 16 active");
    run(k_pass<2, 256>, "barrier only");
    run(k_pass<0, 256, 2>, "full pass, 256 active, 2 accumulators");
    run(k_pass<0, 16, 2>, "full pass, 16 active, 2 accumulators");
    auto runw = [&](auto kern, const char* name) {
        for (int rep = 0; rep < 2; ++rep) {
            kern<<<1, 32>>>(out, cyc, P);
            cudaDeviceSynchronize();
        }
        printf("%-40s %.1f cyc/pass\n", name, (double)cyc[0] / P);
    };
    runw(k_pass<3, 32>, "one warp, syncwarp, 32 active");
    runw(k_pass<3, 16>, "one warp, syncwarp, 16 active");
    runw(k_pass<0, 32>, "one warp, syncthreads, 32 active");
    run(k_pass<1, 16, 2>, "no barrier, 16 active, 2 accumulators");
    return 0;
}
