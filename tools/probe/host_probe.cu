// Host cost of the fused-conv launch ingredients (diagnostics; run on the GPU box).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>

struct Maps { CUtensorMap a, b, c, d; };
__global__ void empty_kernel(int x, const __grid_constant__ Maps m) {}
__global__ void empty_plain(int x) {}

static double now_us() {
    return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main() {
    cudaFree(0);
    void* buf; cudaMalloc(&buf, 64 << 20);
    cudaStream_t st; cudaStreamCreate(&st);
    PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
    PFN_cuTensorMapEncodeIm2col_v12000 enc2 = nullptr;
    cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", (void**)&enc2, cudaEnableDefault, &q);
    CUtensorMap m;
    const int N = 2000;
    double t0 = now_us();
    for (int i = 0; i < N; ++i) {
        cuuint64_t dims[2] = {640, 64}; cuuint64_t strides[1] = {640 * 2};
        cuuint32_t box[2] = {64, 64}; cuuint32_t es[2] = {1, 1};
        enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    printf("encode tiled      %.2f us\n", (now_us() - t0) / N);
    t0 = now_us();
    for (int i = 0; i < N; ++i) {
        cuuint64_t dims[4] = {64, 56, 56, 1}; cuuint64_t strides[3] = {128, 128 * 56, 128 * 56 * 56};
        int lo[2] = {-1, -1}, hi[2] = {-1, -1}; cuuint32_t es[4] = {1, 1, 1, 1};
        enc2(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, buf, dims, strides, lo, hi, 64, 128, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    printf("encode im2col     %.2f us\n", (now_us() - t0) / N);
    Maps mm{m, m, m, m};
    for (int rep = 0; rep < 2; ++rep) {
        cudaDeviceSynchronize();
        t0 = now_us();
        for (int i = 0; i < N; ++i) empty_plain<<<148, 192, 0, st>>>(i);
        printf("launch plain      %.2f us\n", (now_us() - t0) / N);
        cudaDeviceSynchronize();
        t0 = now_us();
        for (int i = 0; i < N; ++i) {
            cudaLaunchConfig_t cfg{}; cfg.gridDim = dim3(148); cfg.blockDim = dim3(192); cfg.stream = st;
            cudaLaunchAttribute attr[1]; attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = 2; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
            cfg.attrs = attr; cfg.numAttrs = 1;
            cudaLaunchKernelEx(&cfg, empty_kernel, i, mm);
        }
        printf("launchEx cluster  %.2f us\n", (now_us() - t0) / N);
        cudaDeviceSynchronize();
        cudaEvent_t ev; cudaEventCreate(&ev);
        t0 = now_us();
        for (int i = 0; i < N; ++i) cudaEventRecord(ev, st);
        printf("event record      %.2f us\n", (now_us() - t0) / N);
        t0 = now_us();
        for (int i = 0; i < N; ++i) cudaGetLastError();
        printf("getlasterror      %.2f us\n", (now_us() - t0) / N);
        cudaDeviceSynchronize();
        // device-side gap: two events around a launch from an idle GPU
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        float acc = 0; 
        for (int i = 0; i < 50; ++i) {
            cudaDeviceSynchronize();
            cudaEventRecord(e0, st); empty_plain<<<148, 192, 0, st>>>(i); cudaEventRecord(e1, st);
            cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); acc += ms;
        }
        printf("idle GPU: event->empty kernel->event  %.2f us\n", acc / 50 * 1e3);
    }
    return 0;
}
