// Microbenchmark (diagnostics only): issue rate of tcgen05.mma kind::f16, M = 128, for
// N in {64, 128, 256}, A from shared memory (SS) or from TMEM (TS), optionally with 4
// warps streaming tcgen05.ld (an epilogue) or tcgen05.st (A producers) at the same time.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2407_10730_b200/csrc \
//        mma_rate.cu -o mma_rate -lcuda
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include "sm100_ptx.cuh"

using namespace cb;

constexpr int ITER = 4096;
__device__ int g_rand = 0;

template <int TS, int N, int SIDE>  // SIDE: 0 none, 1 tcgen05.ld loop, 2 tcgen05.st loop
__global__ void __launch_bounds__(192, 1) mma_rate(unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* a_s = smem;             // 128 x 128 B
    uint8_t* b_s = smem + 16384;     // N x 128 B
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 16384 + 256 * 128);
    uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 4);
    volatile uint32_t* done = slot + 1;
    for (int i = threadIdx.x; i < (16384 + N * 128) / 4; i += blockDim.x)  // random bf16 in [0.5, 1) or zeros
        reinterpret_cast<uint32_t*>(smem)[i] = g_rand ? (((uint32_t)i * 2654435761u) & 0x007f007fu) | 0x3f003f00u : 0u;
    const int warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        ptx::mbar_init(bar, 1); ptx::mbar_init(bar + 2, 1); ptx::mbar_init(bar + 3, 1);
        ptx::mbar_arrive(bar + 3);  // phase 0 complete: waits on it return at once
        *done = 0; ptx::fence_mbar_init();
    }
    ptx::fence_proxy_async_smem();
    if (warp == 5) ptx::tmem_alloc(slot, 512);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tm = *slot;
    if (warp == 5) {
        const uint32_t leader = ptx::elect_one();
        const uint32_t idesc = ptx::idesc_f32acc<true>(128, N);
        const uint64_t da = ptx::sdesc_k_sw128(ptx::smem_u32(a_s));
        const uint64_t db = ptx::sdesc_k_sw128(ptx::smem_u32(b_s));
        const uint32_t a_tm = tm + 256 + 128;  // A columns (TS) after D (N <= 256)
        __syncwarp();
        long long t0 = clock64();
        if (leader) {
            for (int j = 0; j < ITER; ++j) {
                const uint64_t off = (uint64_t)((j & 3) * 2);
                if (TS) ptx::umma_ts_bf16(tm, a_tm + (j & 3) * 8, db + off, idesc, j > 0);
                else ptx::umma<true>(tm, da + off, db + off, idesc, j > 0);
                if (SIDE == 5 && j % 6 == 5) ptx::umma_commit(bar + 2);  // K8: a commit per chunk
                if (SIDE == 6 && j % 6 == 5) {  // + K8's per-chunk wait on a ready barrier and fence
                    ptx::umma_commit(bar + 2);
                    ptx::mbar_wait(bar + 3, 0);
                    ptx::tc_fence_after();
                }
            }
            ptx::umma_commit(bar);
        }
        __syncwarp();
        ptx::mbar_wait(bar, 0);
        long long t1 = clock64();
        if (leader) { *done = 1; if (blockIdx.x == 0) out[0] = (unsigned long long)(t1 - t0); atomicAdd(out + 1, (unsigned long long)(t1 - t0)); }
    } else if (warp < 4 && SIDE) {
        uint32_t r[32] = {};
        unsigned long long n = 0;
        const uint32_t lane_base = tm + ((uint32_t)(warp * 32) << 16);
        while (!*done) {
            if (SIDE == 3) {
                const uint32_t base = ptx::smem_u32(a_s) + 4 * (threadIdx.x & 31);
#pragma unroll
                for (int q = 0; q < 32; ++q) {
                    uint32_t v;
                    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(base + 128 * q));
                    r[q] ^= v;
                }
            } else if (SIDE == 4) {
                const uint32_t base = ptx::smem_u32(b_s) + 16384 + 4 * (threadIdx.x & 31);
#pragma unroll
                for (int q = 0; q < 32; ++q) asm volatile("st.shared.u32 [%0], %1;" ::"r"(base + 128 * (q & 7)), "r"(r[q]));
            } else if (SIDE == 1) {
                ptx::tmem_ld_32x32b_x32(lane_base + (n & 1) * 32, r);
                ptx::tmem_ld_wait();
            } else {
                ptx::tmem_st_32x32b_x32(lane_base + 256 + 128 + 64 + (n & 1) * 32, r);
                ptx::tmem_st_wait();
            }
            ++n;
        }
        if (threadIdx.x == 0) atomicAdd(out + 2 + 0 * blockIdx.x, n);
        if (r[0] == 0x12345u) out[3] = r[1];
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 5) { ptx::tc_fence_after(); ptx::tmem_dealloc(tm, 512); }
}

template <int TS, int N, int SIDE>
void run(unsigned long long* d) {
    cudaMemset(d, 0, 32);
    auto k = mma_rate<TS, N, SIDE>;
    const int smem = 1024 + 16384 + 256 * 128 + 64;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k<<<148, 192, smem>>>(d);
    k<<<148, 192, smem>>>(d + 0);
    cudaMemset(d, 0, 32);
    k<<<148, 192, smem>>>(d);
    unsigned long long h[4];
    cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
    cudaError_t e = cudaGetLastError();
    const double cyc = (double)h[1] / 148 / ITER;
    const double side_bytes = SIDE ? (double)h[2] * 16384.0 / (double)h[1] : 0;  // per SM per cycle
    printf("%s N=%3d side=%s  cycles/MMA %.1f  (block0 %.1f)  floor %d  side B/cyc %.1f  %s\n", TS ? "TS" : "SS", N,
           SIDE == 0 ? "none" : SIDE == 1 ? "ld  " : SIDE == 2 ? "st  " : SIDE == 3 ? "LDS " : SIDE == 4 ? "STS " : SIDE == 5 ? "cmt " : "fnc ", cyc, (double)h[0] / ITER, 128 * N / 256, side_bytes,
           e == cudaSuccess ? "" : cudaGetErrorString(e));
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 64);
    run<0, 64, 0>(d); run<1, 64, 0>(d);
    run<0, 128, 0>(d); run<1, 128, 0>(d);
    run<0, 256, 0>(d); run<1, 256, 0>(d);
    run<1, 64, 1>(d); run<1, 64, 2>(d);
    run<1, 128, 1>(d); run<1, 128, 2>(d);
    run<0, 64, 1>(d); run<0, 64, 2>(d);
    run<1, 64, 3>(d); run<1, 64, 4>(d); run<1, 128, 3>(d); run<0, 64, 3>(d);
    run<1, 256, 5>(d); run<1, 64, 5>(d); run<1, 256, 6>(d); run<1, 64, 6>(d);
    run<1, 256, 1>(d); run<1, 256, 2>(d);
    int one = 1;
    cudaMemcpyToSymbol(g_rand, &one, sizeof(int));
    printf("random operands:\n");
    run<0, 256, 0>(d); run<1, 256, 0>(d); run<1, 256, 2>(d); run<1, 128, 0>(d); run<1, 64, 0>(d);
    return 0;
}
