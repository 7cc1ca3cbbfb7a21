// Microbenchmark (tuning aid): per-kernel time of a captured CUDA graph of N
// dependent small kernels, plain stream order vs programmatic dependent
// launch (PDL: launch attribute + griddepcontrol.wait / launch_dependents).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_pdl tools/ubench_pdl.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int PDL>
__global__ void k_step(double* x, int n)
{
    if (PDL) asm volatile("griddepcontrol.wait;" ::: "memory");
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) x[i] = x[i] * 0.5 + 1.0;
    if (PDL == 2) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

int main()
{
    const int n = 1 << 18, N = 200;
    double* x;
    cudaMalloc(&x, n * sizeof(double));
    cudaMemset(x, 0, n * sizeof(double));
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int blocks : {148, 1024}) {
        for (int mode = 0; mode < 3; ++mode) {
            cudaGraph_t g;
            cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
            for (int k = 0; k < N; ++k) {
                cudaLaunchAttribute at{};
                at.id = cudaLaunchAttributeProgrammaticStreamSerialization;
                at.val.programmaticStreamSerializationAllowed = 1;
                cudaLaunchConfig_t cfg{};
                cfg.gridDim = dim3(blocks);
                cfg.blockDim = dim3(256);
                cfg.stream = s;
                cfg.attrs = &at;
                cfg.numAttrs = mode ? 1 : 0;
                const int nn = blocks * 256 < n ? blocks * 256 : n;
                if (mode == 0) cudaLaunchKernelEx(&cfg, k_step<0>, x, nn);
                else if (mode == 1) cudaLaunchKernelEx(&cfg, k_step<1>, x, nn);
                else cudaLaunchKernelEx(&cfg, k_step<2>, x, nn);
            }
            cudaStreamEndCapture(s, &g);
            cudaGraphExec_t ge;
            cudaGraphInstantiate(&ge, g, 0);
            for (int r = 0; r < 3; ++r) cudaGraphLaunch(ge, s);
            cudaEventRecord(e0, s);
            for (int r = 0; r < 10; ++r) cudaGraphLaunch(ge, s);
            cudaEventRecord(e1, s);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            printf("blocks %4d mode %d (%s): %.2f us per kernel\n", blocks, mode,
                   mode == 0 ? "plain" : mode == 1 ? "PDL wait" : "PDL wait+trigger", 1e3 * ms / (10 * N));
            cudaGraphExecDestroy(ge);
            cudaGraphDestroy(g);
        }
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
