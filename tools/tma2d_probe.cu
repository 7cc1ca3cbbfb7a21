// TMA 2-D tile probe (tuning aid): loads 34 x 18 FP64 boxes (a 32 x 16 tile plus
// a one-node halo, negative and past-the-end coordinates zero-filled) of a
// 1023 x 1023 row-major field with cp.async.bulk.tensor.2d and checks them
// against the field. Kernel written the way CUTLASS's SM90_TMA_LOAD_2D issues it
// (map as a __grid_constant__ parameter, mbarrier init + fence, one elected thread).
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tools/tma2d_probe tools/tma2d_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

constexpr int BX = 34, BY = 18; // box: 34 doubles (272 B, a 16-byte multiple) x 18 rows

__constant__ CUtensorMap c_tm;
__global__ void k_tile(const __grid_constant__ CUtensorMap tm, int n, double* out, int* bad, const CUtensorMap* gtm, int where, int xsc, int xtra)
{
    const unsigned long long desc = where == 0 ? reinterpret_cast<unsigned long long>(&tm)
                                  : where == 1 ? reinterpret_cast<unsigned long long>(gtm)
                                               : reinterpret_cast<unsigned long long>(&c_tm);
    __shared__ __align__(128) double buf[BY][BX];
    __shared__ __align__(8) unsigned long long bar;
    const unsigned sb = (unsigned)__cvta_generic_to_shared(&buf[0][0]);
    const unsigned bb = (unsigned)__cvta_generic_to_shared(&bar);
    const int x0 = blockIdx.x * 32 - 1, y0 = blockIdx.y * 16 - 1;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bb) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bb), "r"(BX * BY * 8) : "memory");
        if (xtra & 1) asm volatile("prefetch.tensormap [%0];" ::"l"(desc) : "memory");
        if (xtra & 2) asm volatile("fence.proxy.tensormap::generic.acquire.gpu [%0], 128;" ::"l"(desc) : "memory");
        if (xtra & 4)
            asm volatile("cp.async.bulk.tensor.2d.shared::cta.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                         ::"r"(sb), "l"(desc), "r"(x0 * xsc), "r"(y0), "r"(bb)
                         : "memory");
        else
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                         ::"r"(sb), "l"(desc), "r"(x0 * xsc), "r"(y0), "r"(bb)
                         : "memory");
    }
    asm volatile("{\n .reg .pred p;\n TW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra TW_%=;\n}" ::"r"(bb)
                 : "memory");
    for (int i = threadIdx.x; i < BX * BY; i += blockDim.x) {
        const int ty = i / BX, tx = i % BX, gx = x0 + tx, gy = y0 + ty;
        const double want = (gx >= 0 && gx < n && gy >= 0 && gy < n) ? (double)gy * n + gx : 0.0;
        if (buf[ty][tx] != want) atomicAdd(bad, 1);
    }
    if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x < 4) out[threadIdx.x] = buf[1][1 + threadIdx.x];
}

int main()
{
    const int n = 1023;
    double *x, *out;
    int* bad;
    cudaMalloc(&x, (size_t)n * n * 8);
    cudaMalloc(&out, 64);
    cudaMalloc(&bad, 4);
    cudaMemset(bad, 0, 4);
    std::vector<double> h((size_t)n * n);
    for (size_t i = 0; i < h.size(); ++i) h[i] = (double)i;
    cudaMemcpy(x, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    CUtensorMap tm;
    cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)n}, strides[1] = {(cuuint64_t)n * 8};
    cuuint32_t box[2] = {BX, BY}, es[2] = {1, 1};
    // the row pitch of a 1023-wide FP64 field (8184 B) is not a 16-byte multiple:
    // TMA needs 16-byte strides, so probe with a padded pitch of 1024.
    double* xp;
    cudaMalloc(&xp, (size_t)n * 1024 * 8);
    cudaMemcpy2D(xp, 1024 * 8, x, n * 8, n * 8, n, cudaMemcpyDeviceToDevice);
    strides[0] = 1024 * 8;
    const int where = getenv("TMA_WHERE") ? atoi(getenv("TMA_WHERE")) : 0;
    const int dtv = getenv("TMA_DT") ? atoi(getenv("TMA_DT")) : 0; // 0 f64, 1 i64, 2 u32 (box x2)
    CUtensorMapDataType dt = dtv == 0 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : dtv == 1 ? CU_TENSOR_MAP_DATA_TYPE_INT64 : CU_TENSOR_MAP_DATA_TYPE_UINT32;
    if (dtv == 2) { dims[0] *= 2; box[0] *= 2; }
    CUresult r = cuTensorMapEncodeTiled(&tm, dt, 2, xp, dims, strides, box, es,
                                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                        CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode -> %d\n", (int)r);
    if (r != CUDA_SUCCESS) return 1;
    dim3 grid((n + 31) / 32, (n + 15) / 16);
    CUtensorMap* gtm;
    cudaMalloc(&gtm, sizeof(tm));
    cudaMemcpy(gtm, &tm, sizeof(tm), cudaMemcpyHostToDevice);
    cudaMemcpyToSymbol(c_tm, &tm, sizeof(tm));
    printf("where=%d dt=%d\n", where, dtv);
    if (dtv == 2) { // coordinates in u32 units
        printf("(u32 view: x coords doubled)\n");
    }
    k_tile<<<grid, 128>>>(tm, n, out, bad, gtm, where, dtv == 2 ? 2 : 1, getenv("TMA_X") ? atoi(getenv("TMA_X")) : 0);
    cudaError_t e = cudaDeviceSynchronize();
    int hb = -1;
    double o[4] = {};
    cudaMemcpy(&hb, bad, 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(o, out, 32, cudaMemcpyDeviceToHost);
    printf("tma2d: %s, mismatches %d, tile(0,0) row 0: %g %g %g %g\n", cudaGetErrorString(e), hb, o[0], o[1], o[2], o[3]);
    return (e == cudaSuccess && hb == 0) ? 0 : 2;
}
