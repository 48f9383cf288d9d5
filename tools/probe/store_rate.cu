// Microbenchmark (diagnostics only): global store bandwidth per SM of an NCHW epilogue --
// W warps per SM, each warp writing 128-byte rows (32 lanes x 4 B) of `rows` channel planes
// (plane stride `pitch` floats), STG.32 vs STG.128 (4 consecutive pixels per lane).
#include <cstdio>
#include <cstdint>

template <int VEC>
__global__ void store_rate(float* out, long long pitch, int rows, int reps) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    // CTA b owns pixels [b * 32 * VEC * nw, ...) of every plane
    const long long px0 = ((long long)blockIdx.x * nw + warp) * 32 * VEC;
    float v = lane;
    for (int rep = 0; rep < reps; ++rep)
        for (int r = 0; r < rows; ++r) {
            float* dst = out + (long long)r * pitch + px0;
            if (VEC == 1) dst[lane] = v + r;
            else reinterpret_cast<float4*>(dst)[lane] = make_float4(v, v + 1, v + 2, v + r);
        }
}

template <int VEC>
void run(float* d, int warps, int rows, long long pitch) {
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    const int reps = 4;
    store_rate<VEC><<<148, warps * 32>>>(d, pitch, rows, reps);
    cudaEventRecord(a);
    store_rate<VEC><<<148, warps * 32>>>(d, pitch, rows, reps);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    const double bytes = 148.0 * warps * 32 * VEC * 4 * rows * reps;
    printf("STG.%d warps/SM %2d rows %3d pitch %lld: %.1f us, %.2f TB/s, %.1f B/clk/SM @1.9GHz  %s\n", 32 * VEC, warps, rows,
           pitch, ms * 1e3, bytes / ms / 1e9, bytes / ms / 1e-3 / 148 / 1.9e9, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    float* d;
    const long long pitch = 12544LL * 16;  // plane pitch in floats (> every CTA's range)
    cudaMalloc(&d, (size_t)pitch * 256 * 4);
    for (int w : {4, 8, 16}) { run<1>(d, w, 64, pitch); run<4>(d, w, 64, pitch); }
    run<1>(d, 4, 256, pitch);
    run<1>(d, 4, 64, 12544);
    return 0;
}
