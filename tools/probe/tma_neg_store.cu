// Probe (diagnostics only): does a TMA tensor store accept a box whose start coordinate is
// negative, writing only the in-bounds part?  3-D fp32 tensor {PQ=40, K=4, N=2}, box
// {32, 4, 1}; store at (p = -20, k = 0, n = 1) from a smem tile holding 100 + i in column i.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I../../paper_2407_10730_b200/csrc tma_neg_store.cu -o tma_neg_store -lcuda
#include <cstdio>
#include <cuda.h>
#include <cudaTypedefs.h>
#include "sm100_ptx.cuh"
using namespace cb;

__global__ void k(const __grid_constant__ CUtensorMap m, int p0) {
    __shared__ __align__(128) float buf[4 * 32];
    for (int i = threadIdx.x; i < 128; i += blockDim.x) buf[i] = 100.f + (i % 32);
    ptx::fence_proxy_async_smem();
    __syncthreads();
    if (threadIdx.x == 0) {
        ptx::tma_store_3d(&m, buf, p0, 0, 1);
        ptx::bulk_commit();
        ptx::bulk_wait_all();
    }
}

int main() {
    const int PQ = 40, K = 4, N = 2;
    float* y;
    cudaMalloc(&y, sizeof(float) * PQ * K * N);
    cudaMemset(y, 0, sizeof(float) * PQ * K * N);
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    CUtensorMap m;
    cuuint64_t dims[3] = {PQ, K, N};
    cuuint64_t strides[2] = {PQ * 4, PQ * K * 4};
    cuuint32_t box[3] = {32, 4, 1};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, y, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode %d\n", (int)r);
    for (int p0 : {20, -20}) {
        cudaMemset(y, 0, sizeof(float) * PQ * K * N);
        k<<<1, 128>>>(m, p0);
        cudaError_t e = cudaDeviceSynchronize();
        float h[PQ * K * N];
        cudaMemcpy(h, y, sizeof(h), cudaMemcpyDeviceToHost);
        printf("p0=%d: %s; image 1, channel 0: ", p0, cudaGetErrorString(e));
        for (int i = 0; i < PQ; ++i) printf("%g ", h[PQ * K + i]);
        printf("\n");
        if (e != cudaSuccess) return 1;
    }
    return 0;
}
