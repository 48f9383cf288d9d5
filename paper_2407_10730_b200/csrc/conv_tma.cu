// conv_tma.cu -- K6: the fused implicit-GEMM convolution, TMA-fed, persistent, tcgen05.
//
// Pipeline of one conv (cb_conv_fused):
//   K0  act_split_nhwc  NCHW fp32 -> NHWC (hi, lo) split once per element (pack_kernels.cu)
//   K6  conv_tma_kernel TMA im2col loads of the (hi, lo) activation tiles + tiled TMA loads
//                       of the pre-split, tap-ordered weights; 3 tcgen05 MMAs per K step
//                       (lo*hi, hi*lo, hi*hi) into a TMEM accumulator; NCHW epilogue.
//
// Why TMA im2col: the hardware walks (n, oy, ox) output pixels of the bounding box with
// the conv stride as traversal stride, adds the filter-tap offset and zero-fills every
// out-of-bounds tap, so padding/stride/dilation cost no instructions and each activation
// is split once instead of R*S times (the gather kernel in conv_tc.cu re-splits per tap).
//
// CTA layout (192 threads, persistent over a static tile schedule, 1 CTA / SM):
//   warp 0      TMA producer (one elected lane)
//   warp 1      TMEM allocator (2 x BN columns: double-buffered accumulator) + MMA issuer
//   warps 2..5  epilogue: tcgen05.ld 32 columns at a time -> +bias -> coalesced NCHW stores
//               (lane = pixel, so each store instruction of a warp writes 32 consecutive
//               pixels of one output channel) or fp32 reductions for split-K.
// Barriers: full/empty per smem stage (TMA tx-count / tcgen05.commit), tmem_full /
// tmem_empty per accumulator buffer, so the epilogue of tile i overlaps the MMAs of i+1.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <mutex>

#include "cb_common.cuh"
#include "sm100_ptx.cuh"

namespace cb {

constexpr int TMA_THREADS = 192;
constexpr int TMA_BM = 128;

struct TmaParams {
    Geom g;
    FusedLayout L;
    const float* bias;
    float* out;
    int n_tiles;          // output-channel tiles per group
    int64_t m_tiles;
    int splits;
    int kb_per_split;
    int64_t total_tiles;  // n_tiles * m_tiles * G * splits
    int add_mode;         // 0: store acc + bias, 1: fp32 reduction into out
};

template <int BN, int STAGES, bool BF16>
struct TmaCfg {
    static constexpr int EB = BF16 ? 2 : 4;
    static constexpr int KE = 128 / EB;              // reduction elements per stage
    static constexpr int A_BYTES = TMA_BM * 128;     // one of A_hi / A_lo
    static constexpr int B_BYTES = BN * 128;
    static constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;
    static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 + 256;
    static constexpr uint32_t TMEM_COLS = 2 * BN;
};

__device__ __forceinline__ void decode_tile(const TmaParams& p, int64_t t, int& nt, int64_t& mt,
                                            int& gi, int& ks) {
    nt = (int)(t % p.n_tiles);
    int64_t r = t / p.n_tiles;
    mt = r % p.m_tiles;
    r /= p.m_tiles;
    gi = (int)(r % p.g.G);
    ks = (int)(r / p.g.G);
}

// K-major descriptor of K step kk (32 bytes of reduction) inside one A stage buffer.
__device__ __forceinline__ uint64_t a_desc(uint32_t base, int chunk_bytes, int kk) {
    switch (chunk_bytes) {
        case 128: return ptx::sdesc_k(base + kk * 32, 2, 1024, 16);
        case 64: return ptx::sdesc_k(base + (kk >> 1) * (TMA_BM * 64) + (kk & 1) * 32, 4, 512, 16);
        case 32: return ptx::sdesc_k(base + kk * (TMA_BM * 32), 6, 256, 16);
        default:  // 16-byte chunks: two consecutive boxes form one 32-byte K step
            return ptx::sdesc_k(base + (2 * kk) * (TMA_BM * 16), 0, 128, TMA_BM * 16);
    }
}

template <int BN, int STAGES, bool BF16>
__global__ void __launch_bounds__(TMA_THREADS, 1)
conv_tma_kernel(const __grid_constant__ TmaParams p, const __grid_constant__ CUtensorMap tm_ahi,
                const __grid_constant__ CUtensorMap tm_alo,
                const __grid_constant__ CUtensorMap tm_bhi,
                const __grid_constant__ CUtensorMap tm_blo) {
    using Cfg = TmaCfg<BN, STAGES, BF16>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * Cfg::STAGE_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const Geom& g = p.g;
    const FusedLayout& L = p.L;

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            ptx::mbar_init(&tfull[a], 1);
            ptx::mbar_init(&tempty[a], 128);
        }
        ptx::fence_mbar_init();
    }
    if (warp == 0 && lane == 0) {
        ptx::tma_prefetch_desc(&tm_ahi);
        ptx::tma_prefetch_desc(&tm_alo);
        ptx::tma_prefetch_desc(&tm_bhi);
        ptx::tma_prefetch_desc(&tm_blo);
    }
    if (warp == 1) ptx::tmem_alloc(tmem_slot, Cfg::TMEM_COLS);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        // ================================ TMA producer ==================================
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            constexpr uint32_t tx = 2 * Cfg::A_BYTES + 2 * Cfg::B_BYTES;
            for (int64_t t = blockIdx.x; t < p.total_tiles; t += gridDim.x) {
                int nt, gi, ks;
                int64_t mt;
                decode_tile(p, t, nt, mt, gi, ks);
                const int64_t m0 = mt * TMA_BM;
                const int n0 = (int)(m0 / g.PQ);
                const int rem = (int)(m0 - (int64_t)n0 * g.PQ);
                const int oy0 = rem / g.Q, ox0 = rem - (rem / g.Q) * g.Q;
                const int wc = ox0 * g.sw - g.pw, hc = oy0 * g.sh - g.ph;
                const int brow = gi * g.kpg + nt * BN;
                const int kb0 = ks * p.kb_per_split;
                const int kb1 = min(L.num_kb, kb0 + p.kb_per_split);
                for (int kb = kb0; kb < kb1; ++kb) {
                    ptx::mbar_wait(&empty[stage], phase ^ 1);
                    uint8_t* st = smem + stage * Cfg::STAGE_BYTES;
                    ptx::mbar_arrive_expect_tx(&full[stage], tx);
                    for (int i = 0; i < L.cps; ++i) {
                        const int q = kb * L.cps + i;
                        int c = L.c_alloc, offw = 0, offh = 0;  // past the end: all-OOB zeros
                        if (q < L.total_chunks) {
                            const int tap = q / L.chk;
                            const int cbi = q - tap * L.chk;
                            const int r = tap / g.S, s = tap - (tap / g.S) * g.S;
                            c = gi * g.cpg + cbi * L.cb;
                            offw = s * g.dw;
                            offh = r * g.dh;
                        }
                        const int off = i * TMA_BM * L.chunk_bytes;
                        ptx::tma_load_im2col_4d(st + off, &tm_ahi, &full[stage], c, wc, hc, n0,
                                                (uint16_t)offw, (uint16_t)offh);
                        ptx::tma_load_im2col_4d(st + Cfg::A_BYTES + off, &tm_alo, &full[stage], c,
                                                wc, hc, n0, (uint16_t)offw, (uint16_t)offh);
                    }
                    ptx::tma_load_2d(st + 2 * Cfg::A_BYTES, &tm_bhi, &full[stage], kb * Cfg::KE,
                                     brow);
                    ptx::tma_load_2d(st + 2 * Cfg::A_BYTES + Cfg::B_BYTES, &tm_blo, &full[stage],
                                     kb * Cfg::KE, brow);
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ================================= MMA issuer ===================================
        if (lane == 0) {
            constexpr uint32_t idesc = ptx::idesc_f32acc<BF16>(TMA_BM, BN);
            int stage = 0;
            uint32_t phase = 0;
            int local = 0;
            for (int64_t t = blockIdx.x; t < p.total_tiles; t += gridDim.x, ++local) {
                int nt, gi, ks;
                int64_t mt;
                decode_tile(p, t, nt, mt, gi, ks);
                const int acc = local & 1;
                const uint32_t acc_phase = (local >> 1) & 1;
                ptx::mbar_wait(&tempty[acc], acc_phase ^ 1);
                ptx::tc_fence_after();
                const uint32_t d = tmem_base + acc * BN;
                const int kb0 = ks * p.kb_per_split;
                const int kb1 = min(L.num_kb, kb0 + p.kb_per_split);
                for (int kb = kb0; kb < kb1; ++kb) {
                    ptx::mbar_wait(&full[stage], phase);
                    ptx::tc_fence_after();
                    const uint32_t a_hi = ptx::smem_u32(smem + stage * Cfg::STAGE_BYTES);
                    const uint32_t a_lo = a_hi + Cfg::A_BYTES;
                    const uint32_t b_hi = a_hi + 2 * Cfg::A_BYTES;
                    const uint32_t b_lo = b_hi + Cfg::B_BYTES;
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {
                        const uint64_t dah = a_desc(a_hi, L.chunk_bytes, kk);
                        const uint64_t dal = a_desc(a_lo, L.chunk_bytes, kk);
                        const uint64_t dbh = ptx::sdesc_k_sw128(b_hi + kk * 32);
                        const uint64_t dbl = ptx::sdesc_k_sw128(b_lo + kk * 32);
                        ptx::umma<BF16>(d, dal, dbh, idesc, (kb != kb0 || kk != 0) ? 1u : 0u);
                        ptx::umma<BF16>(d, dah, dbl, idesc, 1);
                        ptx::umma<BF16>(d, dah, dbh, idesc, 1);
                    }
                    ptx::umma_commit(&empty[stage]);
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                ptx::umma_commit(&tfull[acc]);
            }
        }
    } else {
        // ================================== epilogue ===================================
        const int quad = warp & 3;           // TMEM lane quadrant this warp may access
        const int row = quad * 32 + lane;    // pixel row within the tile
        int local = 0;
        for (int64_t t = blockIdx.x; t < p.total_tiles; t += gridDim.x, ++local) {
            int nt, gi, ks;
            int64_t mt;
            decode_tile(p, t, nt, mt, gi, ks);
            const int acc = local & 1;
            const uint32_t acc_phase = (local >> 1) & 1;
            ptx::mbar_wait(&tfull[acc], acc_phase);
            ptx::tc_fence_after();
            const int64_t j = mt * TMA_BM + row;
            const bool jvalid = j < g.npix;
            int64_t obase = 0;
            if (jvalid) {
                const int64_t n = j / g.PQ;
                obase = n * (int64_t)g.K * g.PQ + (j - n * g.PQ);
            }
            const int f_tile0 = nt * BN;
#pragma unroll 1
            for (int c0 = 0; c0 < BN; c0 += 32) {
                if (f_tile0 + c0 >= g.kpg) break;  // warp-uniform
                uint32_t r[32];
                ptx::tmem_ld_32x32b_x32(tmem_base + acc * BN + ((uint32_t)(quad * 32) << 16) + c0,
                                        r);
                ptx::tmem_ld_wait();
                if (jvalid) {
#pragma unroll
                    for (int i = 0; i < 32; ++i) {
                        const int fl = f_tile0 + c0 + i;
                        if (fl < g.kpg) {
                            const int f = gi * g.kpg + fl;
                            float* dst = p.out + obase + (int64_t)f * g.PQ;
                            const float a = __uint_as_float(r[i]);
                            if (p.add_mode)
                                atomicAdd(dst, a);
                            else
                                *dst = a + (p.bias ? __ldg(p.bias + f) : 0.f);
                        }
                    }
                }
            }
            ptx::tc_fence_before();
            ptx::mbar_arrive(&tempty[acc]);
        }
    }

    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem_base, Cfg::TMEM_COLS);
    }
}

// ----------------------------------------------------------------------------------------
// Host side
// ----------------------------------------------------------------------------------------
static PFN_cuTensorMapEncodeIm2col_v12000 im2col_encode_fn() {
    static PFN_cuTensorMapEncodeIm2col_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &ptr, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeIm2col_v12000>(ptr);
    });
    return fn;
}
static PFN_cuTensorMapEncodeTiled_v12000 tiled_encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
    });
    return fn;
}

static int next_pow2(int v) {
    int p = 1;
    while (p < v) p <<= 1;
    return p;
}

FusedLayout fused_layout(const Geom& g, bool bf16) {
    FusedLayout L{};
    L.eb = bf16 ? 2 : 4;
    const int align = 16 / L.eb;      // channels per 16 bytes
    const int maxcb = 128 / L.eb;     // channels per 128-byte row
    L.c_alloc = round_up(g.C, align);
    if (g.G == 1) {
        L.cb = std::min(maxcb, std::max(align, next_pow2(g.C)));
    } else {
        // chunks must not straddle groups: largest power of two dividing cpg
        int cb = maxcb;
        while (cb > align && g.cpg % cb) cb >>= 1;
        L.cb = cb;
    }
    L.chunk_bytes = L.cb * L.eb;
    L.chk = (g.cpg + L.cb - 1) / L.cb;
    L.cps = 128 / L.chunk_bytes;
    L.total_chunks = g.R * g.S * L.chk;
    L.num_kb = (L.total_chunks + L.cps - 1) / L.cps;
    L.kw_pad = L.num_kb * maxcb;
    L.act_elems = (int64_t)g.N * g.HW * L.c_alloc;
    // TMA im2col limits: rank-4 corner offsets in [-128, 127], traversal strides <= 8,
    // 16-bit tap offsets; groups need chunk-aligned group boundaries.
    const int lw = -g.pw, lh = -g.ph;
    const int uw = g.pw - (g.S - 1) * g.dw, uh = g.ph - (g.R - 1) * g.dh;
    bool ok = lw >= -128 && lh >= -128 && uw >= -128 && uh >= -128 && uw <= 127 && uh <= 127;
    ok = ok && g.sh <= 8 && g.sw <= 8 && (g.S - 1) * g.dw < 65536 && (g.R - 1) * g.dh < 65536;
    ok = ok && (g.G == 1 || g.cpg % L.cb == 0);
    ok = ok && (int64_t)g.N * g.HW * L.c_alloc * L.eb < (1LL << 40);
    L.tma = ok ? 1 : 0;
    return L;
}

struct TmaPlan {
    int bn, stages, splits, kb_per_split, n_tiles;
    int64_t m_tiles, total_tiles;
    int grid;
};

static TmaPlan plan_tma(const Geom& g, const FusedLayout& L) {
    TmaPlan pl{};
    const int sms = sm_count();
    pl.m_tiles = ceil_div64(g.npix, TMA_BM);
    int best_bn = 64;
    double best = 1e300;
    for (int bn : {256, 128, 64}) {
        if (bn > 64 && g.kpg <= bn / 2) continue;
        const int64_t tiles = pl.m_tiles * ((g.kpg + bn - 1) / bn) * g.G;
        // persistent: per-SM work = ceil(tiles / sms) tiles of (bn * num_kb) MMA cycles,
        // plus a per-tile fixed cost; wide tiles re-read activations fewer times
        const double per_sm = std::ceil((double)tiles / sms);
        const double cost = per_sm * ((double)bn * L.num_kb + 1500.0);
        if (cost < best * 0.97) {
            best = cost;
            best_bn = bn;
        }
    }
    pl.bn = best_bn;
    pl.n_tiles = (g.kpg + pl.bn - 1) / pl.bn;
    const int64_t tiles = pl.m_tiles * pl.n_tiles * g.G;
    pl.splits = 1;
    if (tiles < sms && L.num_kb >= 4) {
        int want = (int)((sms + tiles - 1) / tiles);
        pl.splits = std::max(1, std::min(want, L.num_kb / 2));
    }
    pl.kb_per_split = (L.num_kb + pl.splits - 1) / pl.splits;
    pl.splits = (L.num_kb + pl.kb_per_split - 1) / pl.kb_per_split;
    pl.total_tiles = tiles * pl.splits;
    pl.stages = pl.bn == 256 ? 2 : (pl.bn == 128 ? 3 : 4);
    pl.grid = (int)std::min<int64_t>(pl.total_tiles, sms);
    return pl;
}

int tma_plan_query(const Geom& g, bool bf16, cb_tile_plan* out) {
    FusedLayout L = fused_layout(g, bf16);
    TmaPlan pl = plan_tma(g, L);
    out->variant = bf16 ? CB_VARIANT_TC3XBF16 : CB_VARIANT_TC3XTF32;
    out->block_m = TMA_BM;
    out->block_n = pl.bn;
    out->block_k = 128 / L.eb;
    out->stages = pl.stages;
    out->splits = pl.splits;
    out->m_tiles = pl.m_tiles;
    out->n_tiles = (int64_t)pl.n_tiles * g.G;
    out->k_blocks = L.num_kb;
    out->ctas = pl.grid;
    return CB_OK;
}

static int make_act_map(CUtensorMap* m, bool bf16, const Geom& g, const FusedLayout& L,
                        const void* base) {
    auto fn = im2col_encode_fn();
    if (!fn) return fail(CB_ERR_CUDA, "cuTensorMapEncodeIm2col unavailable");
    if (reinterpret_cast<uintptr_t>(base) & 15)
        return fail(CB_ERR_MISALIGNED, "activation workspace must be 16-byte aligned");
    cuuint64_t dims[4] = {(cuuint64_t)L.c_alloc, (cuuint64_t)g.W, (cuuint64_t)g.H, (cuuint64_t)g.N};
    cuuint64_t strides[3] = {(cuuint64_t)L.c_alloc * L.eb, (cuuint64_t)g.W * L.c_alloc * L.eb,
                             (cuuint64_t)g.HW * L.c_alloc * L.eb};
    int lower[2] = {-g.pw, -g.ph};
    int upper[2] = {g.pw - (g.S - 1) * g.dw, g.ph - (g.R - 1) * g.dh};
    cuuint32_t estr[4] = {1, (cuuint32_t)g.sw, (cuuint32_t)g.sh, 1};
    CUtensorMapSwizzle sw = L.chunk_bytes == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                            : L.chunk_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                            : L.chunk_bytes == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                                                  : CU_TENSOR_MAP_SWIZZLE_NONE;
    CUresult r = fn(m, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4,
                    const_cast<void*>(base), dims, strides, lower, upper, (cuuint32_t)L.cb,
                    (cuuint32_t)TMA_BM, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        return fail(CB_ERR_CUDA, "cuTensorMapEncodeIm2col failed: " + std::to_string((int)r));
    return CB_OK;
}

static int make_w_map(CUtensorMap* m, bool bf16, const void* w, int rows, int kw_pad, int bn) {
    auto fn = tiled_encode_fn();
    if (!fn) return fail(CB_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    if (reinterpret_cast<uintptr_t>(w) & 15)
        return fail(CB_ERR_MISALIGNED, "packed weights must be 16-byte aligned");
    const int eb = bf16 ? 2 : 4;
    cuuint64_t dims[2] = {(cuuint64_t)kw_pad, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)kw_pad * eb};
    cuuint32_t box[2] = {(cuuint32_t)(128 / eb), (cuuint32_t)bn};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(m, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                    const_cast<void*>(w), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        return fail(CB_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
    return CB_OK;
}

template <int BN, int STAGES, bool BF16>
static int launch_tma_cfg(const TmaParams& prm, int grid, const void* ahi, const void* alo,
                          const void* whi, const void* wlo, cudaStream_t st) {
    using Cfg = TmaCfg<BN, STAGES, BF16>;
    static std::once_flag once;
    static cudaError_t attr_err = cudaSuccess;
    std::call_once(once, [] {
        attr_err = cudaFuncSetAttribute(conv_tma_kernel<BN, STAGES, BF16>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        Cfg::SMEM_BYTES);
    });
    if (attr_err != cudaSuccess)
        return fail(CB_ERR_CUDA, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(attr_err));
    CUtensorMap mah, mal, mwh, mwl;
    int rc;
    if ((rc = make_act_map(&mah, BF16, prm.g, prm.L, ahi))) return rc;
    if ((rc = make_act_map(&mal, BF16, prm.g, prm.L, alo))) return rc;
    if ((rc = make_w_map(&mwh, BF16, whi, prm.g.K, prm.L.kw_pad, BN))) return rc;
    if ((rc = make_w_map(&mwl, BF16, wlo, prm.g.K, prm.L.kw_pad, BN))) return rc;
    conv_tma_kernel<BN, STAGES, BF16>
        <<<grid, TMA_THREADS, Cfg::SMEM_BYTES, st>>>(prm, mah, mal, mwh, mwl);
    return check_launch("conv_tma_kernel");
}

int launch_fill_bias(int64_t images, int K, int PQ, const float* bias, float* y, cudaStream_t st);

// The TMA conv proper (K6), activations already split into the NHWC workspace.
int launch_conv_tma(bool bf16, const Geom& g, const FusedLayout& L, const void* act_hi,
                    const void* act_lo, const void* w_hi, const void* w_lo, const float* bias,
                    float* y, cudaStream_t st) {
    if (g.npix == 0) return CB_OK;
    TmaPlan pl = plan_tma(g, L);
    TmaParams prm{};
    prm.g = g;
    prm.L = L;
    prm.bias = bias;
    prm.out = y;
    prm.n_tiles = pl.n_tiles;
    prm.m_tiles = pl.m_tiles;
    prm.splits = pl.splits;
    prm.kb_per_split = pl.kb_per_split;
    prm.total_tiles = pl.total_tiles;
    prm.add_mode = 0;
    if (pl.splits > 1) {
        int rc = launch_fill_bias(g.N, g.K, g.PQ, bias, y, st);
        if (rc) return rc;
        prm.add_mode = 1;
    }
#define CB_TMA_CASE(BN_, ST_)                                                                  \
    if (pl.bn == BN_ && pl.stages == ST_)                                                      \
        return bf16 ? launch_tma_cfg<BN_, ST_, true>(prm, pl.grid, act_hi, act_lo, w_hi, w_lo, st) \
                    : launch_tma_cfg<BN_, ST_, false>(prm, pl.grid, act_hi, act_lo, w_hi, w_lo, st);
    CB_TMA_CASE(256, 2)
    CB_TMA_CASE(128, 3)
    CB_TMA_CASE(64, 4)
#undef CB_TMA_CASE
    return fail(CB_ERR_UNSUPPORTED, "no TMA tile configuration");
}

}  // namespace cb
