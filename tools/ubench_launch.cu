// Microbenchmark (tuning aid): host enqueue cost and back-to-back device time
// of a plain launch vs a 16-CTA non-portable cluster launch (cudaLaunchKernelEx).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_launch tools/ubench_launch.cu
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_empty(int* p) { if (p && threadIdx.x == 1023) p[0] = 1; }
__global__ void __launch_bounds__(256, 1) k_cl(int* p, int big) {
    extern __shared__ double sm[];
    if (p && threadIdx.x == 1023) p[0] = (int)sm[big];
}

int main()
{
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    cudaFuncSetAttribute(k_cl, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    const int smem = 200 * 1024;
    cudaFuncSetAttribute(k_cl, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int N = 2000;
    auto bench = [&](const char* name, auto fn) {
        for (int i = 0; i < 50; ++i) fn();
        cudaStreamSynchronize(s);
        auto t0 = std::chrono::steady_clock::now();
        cudaEventRecord(e0, s);
        for (int i = 0; i < N; ++i) fn();
        cudaEventRecord(e1, s);
        auto t1 = std::chrono::steady_clock::now();
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("%-34s host enqueue %.2f us/launch, device %.2f us/launch\n", name,
               std::chrono::duration<double, std::micro>(t1 - t0).count() / N, 1e3 * ms / N);
    };
    bench("plain <<<256,256>>>", [&] { k_empty<<<256, 256, 0, s>>>(nullptr); });
    cudaLaunchAttribute at{};
    at.id = cudaLaunchAttributeClusterDimension;
    at.val.clusterDim.x = 16; at.val.clusterDim.y = 1; at.val.clusterDim.z = 1;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(16); cfg.blockDim = dim3(256); cfg.dynamicSmemBytes = smem; cfg.stream = s;
    cfg.attrs = &at; cfg.numAttrs = 1;
    bench("cluster 16 x 256, 200 KB smem", [&] { cudaLaunchKernelEx(&cfg, k_cl, (int*)nullptr, 0); });
    cfg.numAttrs = 0;
    bench("no cluster 16 x 256, 200 KB smem", [&] { cudaLaunchKernelEx(&cfg, k_cl, (int*)nullptr, 0); });
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
