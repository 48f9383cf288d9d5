// Probe (diagnostics only): DRAM read rate of cfg4's NCHW input (N=128, C=256, 14x14 fp32,
// 25.7 MB) with K0's access pattern -- blocks of 128 flattened pixels x 64 channels, 512-byte
// runs per channel plane (planes 784 bytes apart) -- against whole-image blocks that read
// 64 contiguous planes (50 KB runs).  Each block sums its floats (no writes); L2 flushed
// between launches.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 read_pattern.cu -o read_pattern
#include <cstdio>
#include <cuda_runtime.h>

constexpr int N = 128, C = 256, HW = 196;

__global__ void k0_pattern(const float* __restrict__ x, float* out) {  // grid (196, 4), 256 thr
    const long j0 = (long)blockIdx.x * 128;
    const int c0 = blockIdx.y * 64, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const long jg = j0 + 4 * lane;
    const long n = jg / HW;
    const float* xg = x + n * (long)C * HW + (jg - n * HW);
    float acc = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(xg + (long)(c0 + warp + 8 * i) * HW));
        acc += v.x + v.y + v.z + v.w;
    }
    if (acc == 1234.5f) out[0] = acc;
}

__global__ void image_pattern(const float* __restrict__ x, float* out) {  // grid (128, 4), 256 thr
    const float* base = x + ((long)blockIdx.x * C + blockIdx.y * 64) * HW;  // 64 planes, contiguous
    constexpr int n4 = 64 * HW / 4;  // 3136 float4
    float acc = 0.f;
    for (int i = threadIdx.x; i < n4; i += 256 * 4) {
        float4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
            v[u] = i + u * 256 < n4 ? __ldg(reinterpret_cast<const float4*>(base) + i + u * 256) : make_float4(0, 0, 0, 0);
#pragma unroll
        for (int u = 0; u < 4; ++u) acc += v[u].x + v[u].y + v[u].z + v[u].w;
    }
    if (acc == 1234.5f) out[0] = acc;
}

int main() {
    float *x, *out, *flush;
    const size_t bytes = (size_t)N * C * HW * 4;
    cudaMalloc(&x, bytes);
    cudaMalloc(&out, 64);
    cudaMalloc(&flush, 256 << 20);
    cudaMemset(x, 0, bytes);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaMemset(flush, 1, 256 << 20);
    for (int rep = 0; rep < 3; ++rep) {
        for (int kind = 0; kind < 2; ++kind) {
            // evict x with clean lines: read 256 MB (after the one-time write above)
            image_pattern<<<dim3(256 * 1024 * 1024 / (C * HW * 4) / 4 * 4, 4), 256>>>(flush, out);
            cudaDeviceSynchronize();
            cudaEventRecord(e0);
            if (kind == 0)
                k0_pattern<<<dim3(N * HW / 128, 4), 256>>>(x, out);
            else
                image_pattern<<<dim3(N, 4), 256>>>(x, out);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            printf("%s: %.2f us  %.2f TB/s\n", kind ? "whole-image blocks" : "K0 pattern", ms * 1e3, bytes / (ms * 1e-3) / 1e12);
        }
    }
    return 0;
}
