// Microbenchmark (tuning aid): FP64 dependent-chain latencies on the device.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_fp64 tools/ubench_fp64.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_chain(double* out, long long* cyc, double a, double b, int n)
{
    double x = threadIdx.x * 1e-3;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
        x = fma(x, a, b);
        x = fma(x, a, b);
        x = fma(x, a, b);
        x = fma(x, a, b);
    }
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void k_mulchain(double* out, long long* cyc, double a, int n)
{
    double x = threadIdx.x * 1e-3 + 1.0;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
        x = x * a;
        x = x * a;
        x = x * a;
        x = x * a;
    }
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

// LDS -> DFMA -> STS dependent chain through shared memory
__global__ void k_ldsfma(double* out, long long* cyc, double a, int n)
{
    __shared__ double s[64];
    if (threadIdx.x < 64) s[threadIdx.x] = threadIdx.x;
    __syncthreads();
    int idx = threadIdx.x & 31;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
        double v = s[idx];
        s[idx] = fma(v, a, 1.0);
    }
    long long t1 = clock64();
    out[threadIdx.x] = s[idx];
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void k_bar(long long* cyc, int n)
{
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

int main()
{
    double* out;
    long long* cyc;
    cudaMalloc(&out, 4096 * sizeof(double));
    cudaMallocManaged(&cyc, sizeof(long long));
    const int n = 4096;
    for (int rep = 0; rep < 2; ++rep) {
        k_chain<<<1, 32>>>(out, cyc, 0.999, 1e-3, n);
        cudaDeviceSynchronize();
        if (rep) printf("DFMA dependent latency: %.2f cyc\n", (double)cyc[0] / (4.0 * n));
        k_mulchain<<<1, 32>>>(out, cyc, 0.999, n);
        cudaDeviceSynchronize();
        if (rep) printf("DMUL dependent latency: %.2f cyc\n", (double)cyc[0] / (4.0 * n));
        k_ldsfma<<<1, 32>>>(out, cyc, 0.999, n);
        cudaDeviceSynchronize();
        if (rep) printf("LDS->DFMA->STS chain: %.2f cyc/iter\n", (double)cyc[0] / n);
        for (int nt : {32, 256, 1024}) {
            k_bar<<<1, nt>>>(cyc, n);
            cudaDeviceSynchronize();
            if (rep) printf("__syncthreads (%d thr): %.2f cyc\n", nt, (double)cyc[0] / n);
        }
    }
    return 0;
}
