// Tuning aid: how many thread-block clusters of a given size (one CTA per SM:
// 256 threads, ~220 KB of shared memory) can be resident at once.
//   nvcc -arch=sm_100a -o tools/cluster_occ tools/cluster_occ.cu && tools/cluster_occ
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(256, 1) k(int* p) { extern __shared__ double sm[]; if (p) p[0] = (int)sm[0]; }
int main()
{
    cudaDeviceProp pr;
    cudaGetDeviceProperties(&pr, 0);
    printf("%s: %d SMs\n", pr.name, pr.multiProcessorCount);
    cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int smem : {220 * 1024, 100 * 1024, 48 * 1024}) {
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        for (int cs : {16, 12, 10, 8, 6, 4, 2}) {
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3(cs * 64);
            cfg.blockDim = dim3(256);
            cfg.dynamicSmemBytes = smem;
            cudaLaunchAttribute at{};
            at.id = cudaLaunchAttributeClusterDimension;
            at.val.clusterDim.x = cs;
            at.val.clusterDim.y = at.val.clusterDim.z = 1;
            cfg.attrs = &at;
            cfg.numAttrs = 1;
            int n = -1;
            cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k, &cfg);
            printf("smem %3d KB cluster %2d: max active clusters %d (%d SMs) %s\n", smem / 1024, cs, n,
                   n * cs, e == cudaSuccess ? "" : cudaGetErrorString(e));
            cudaGetLastError();
        }
    }
    return 0;
}
