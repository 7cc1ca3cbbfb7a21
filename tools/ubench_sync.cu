// Microbenchmark (tuning aid): cost of cluster barriers, block barriers and
// a dependent FP64 smem update chain on this B200, with the GPU warmed up.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ubench tools/ubench_sync.cu
#include <cooperative_groups.h>
#include <cstdio>

namespace cg = cooperative_groups;

__global__ void k_cluster_sync(int iters, unsigned long long* out)
{
    cg::cluster_group cl = cg::this_cluster();
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) cl.sync();
    unsigned long long t1 = clock64();
    if (threadIdx.x == 0 && cl.block_rank() == 0) out[0] = t1 - t0;
}

__global__ void k_cluster_arrive_wait(int iters, unsigned long long* out)
{
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");
        asm volatile("barrier.cluster.wait.aligned;\n" ::: "memory");
    }
    unsigned long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = t1 - t0;
}

__global__ void k_block_sync(int iters, unsigned long long* out)
{
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) __syncthreads();
    unsigned long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = t1 - t0;
}

__global__ void k_named_sync(int iters, int nthreads, unsigned long long* out)
{
    if (threadIdx.x >= nthreads) return;
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
    unsigned long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = t1 - t0;
}

__global__ void k_gs_chain(int iters, unsigned long long* out, double* sink)
{
    __shared__ double x[1024 + 64];
    __shared__ double c[4 * 1024];
    for (int i = threadIdx.x; i < 1024 + 64; i += blockDim.x) x[i] = 1.0 + i * 1e-3;
    for (int i = threadIdx.x; i < 4 * 1024; i += blockDim.x) c[i] = 1e-2 * (i % 7);
    __syncthreads();
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        const int l = threadIdx.x + 32;
        double acc = x[l];
#pragma unroll
        for (int d = 0; d < 9; ++d) {
            if (d == 4) continue;
            acc -= c[(d & 3) * 1024 + threadIdx.x] * x[l + (d % 3 - 1) + 8 * (d / 3 - 1)];
        }
        x[l] = acc * 0.25;
        __syncthreads();
    }
    unsigned long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = t1 - t0;
    if (threadIdx.x == 0) sink[blockIdx.x] = x[40];
}

template <typename K, typename... A>
double run_cluster(K kern, int cs, int threads, int iters, A... args)
{
    unsigned long long* d;
    cudaMalloc(&d, 8);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(cs);
    cfg.blockDim = dim3(threads);
    cudaLaunchAttribute at{};
    at.id = cudaLaunchAttributeClusterDimension;
    at.val.clusterDim.x = cs;
    at.val.clusterDim.y = 1;
    at.val.clusterDim.z = 1;
    cfg.attrs = &at;
    cfg.numAttrs = 1;
    cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int w = 0; w < 3; ++w) cudaLaunchKernelEx(&cfg, kern, iters, d, args...);
    cudaDeviceSynchronize();
    unsigned long long h = 0;
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    cudaFree(d);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
    return (double)h / iters;
}

int main()
{
    // warm the clocks
    double* sink;
    cudaMalloc(&sink, 1 << 20);
    unsigned long long* d;
    cudaMalloc(&d, 8);
    for (int i = 0; i < 200; ++i) k_gs_chain<<<148, 1024>>>(2000, d, sink);
    cudaDeviceSynchronize();
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("clock rate attr %d kHz\n", clk);
    const int it = 2000;
    for (int cs : {2, 4, 8, 16}) {
        printf("cluster.sync       cs=%2d threads=1024: %.0f cycles\n", cs,
               run_cluster(k_cluster_sync, cs, 1024, it));
        printf("arrive.relaxed+wait cs=%2d threads=1024: %.0f cycles\n", cs,
               run_cluster(k_cluster_arrive_wait, cs, 1024, it));
        printf("cluster.sync       cs=%2d threads=256 : %.0f cycles\n", cs,
               run_cluster(k_cluster_sync, cs, 256, it));
    }
    unsigned long long h;
    k_block_sync<<<1, 1024>>>(it, d);
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("__syncthreads 1024: %.0f cycles\n", (double)h / it);
    k_block_sync<<<1, 256>>>(it, d);
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("__syncthreads 256: %.0f cycles\n", (double)h / it);
    for (int nt : {64, 256}) {
        k_named_sync<<<1, 1024>>>(it, nt, d);
        cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        printf("bar.sync %d of 1024: %.0f cycles\n", nt, (double)h / it);
    }
    k_gs_chain<<<1, 1024>>>(it, d, sink);
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("GS node update + syncthreads (1024 thr): %.0f cycles\n", (double)h / it);
    k_gs_chain<<<1, 256>>>(it, d, sink);
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("GS node update + syncthreads (256 thr): %.0f cycles\n", (double)h / it);
    return 0;
}
