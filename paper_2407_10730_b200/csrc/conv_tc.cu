// conv_tc.cu -- tcgen05 implicit-GEMM convolution / GEMM with a 3-product split
// (3xTF32 or 3xBF16) for fp32-grade results on the 5th-generation tensor cores.
//
// One kernel template serves three reference call sites:
//   * conv_fused       (SRC_CONV):   the whole conv, activations gathered from NCHW
//                                    (implicit im2col, no workspace)         -> K6
//   * the im2col GEMM  (SRC_MATRIX): gemm(wmat, cols) of algos.py:142-182,203-208 -> K4
//   * the SConv GEMM   (SRC_MATRIX, a chunk's slices): wmat[f0:f1] @ pmat of algos.py:326-330 -> K4
//
// GEMM mapping (per group gi):
//   M  = pixels j (128 per CTA tile, one TMEM lane each)
//   N  = output channels f (BN per tile: 64 / 128 / 256 TMEM columns, fp32)
//   K  = reduction k = (c, ky, kx) in OIHW order, so the weights need no reorder.
//
// Warp roles (192 threads, one CTA tile per CTA):
//   warps 0-3  activation producers: each thread owns one pixel row of the 128 x BK tile,
//              gathers it with predicated loads (stride / padding / dilation / groups),
//              splits every value into (hi, lo) and writes both 128B-swizzled K-major
//              rows to shared memory; after the main loop the same warps are the
//              epilogue (tcgen05.ld -> +bias -> coalesced NCHW stores or fp32 reductions).
//   warp  4    TMA producer: weight hi/lo tiles (pre-split by K3) via cp.async.bulk.tensor.
//   warp  5    TMEM allocator + single-thread MMA issuer: per BK slice, for each UMMA_K
//              step, three MMAs  A_lo*B_hi, A_hi*B_lo, A_hi*B_hi  into one TMEM accumulator.
//
// Pipeline: STAGES-deep smem ring with full (128 producer arrivals + TMA tx bytes) and
// empty (tcgen05.commit) mbarriers; one tmem_full barrier hands the accumulator to the
// epilogue.  Split-K (grid.z) accumulates with fp32 reductions into a bias-initialised
// output, exactly the "caller pre-initialises c_out" contract of gemm (algos.py:149-158).
#include <cudaTypedefs.h>

#include <mutex>

#include "cb_common.cuh"
#include "sm100_ptx.cuh"

namespace cb {

struct TcParams {
    Geom g;
    PixMap pm;
    const float* src;   // x (SRC_CONV), cols / b matrix / SConv slices (SRC_MATRIX)
    const float* bias;  // (K,) or null; only added in store mode
    float* out;
    int num_kb;         // k blocks of BK over kdim
    int kb_per_split;   // k blocks per grid.z slice
    int n_tiles;        // output-channel tiles per group
    int add_mode;       // 0: out = acc + bias, 1: out += acc (fp32 reduction)
};

constexpr int TC_THREADS = 192;
constexpr int TC_BM = 128;

template <int BN, int STAGES, bool BF16>
struct TcCfg {
    static constexpr int EB = BF16 ? 2 : 4;         // bytes per operand element
    static constexpr int BK = 128 / EB;             // k per stage: one 128-byte swizzle row
    static constexpr int UK = 32 / EB;              // k per tcgen05.mma
    static constexpr int A_BYTES = TC_BM * 128;     // one of A_hi / A_lo
    static constexpr int B_BYTES = BN * 128;        // one of B_hi / B_lo
    static constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;
    static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
    static_assert(BN == 64 || BN == 128 || BN == 256, "BN");
};

// Gather one BK-wide k slice of the pixel row owned by this thread.
template <int BK>
__device__ __forceinline__ void gather_row(const TcParams& p, int gi, int k0, bool jvalid,
                                           const float* __restrict__ xb, int iy0, int ix0,
                                           int64_t lbase, int64_t lstride, float (&v)[BK]) {
    const Geom& g = p.g;
    if (p.pm.src_mode == SRC_CONV) {
        int c = k0 / g.RS;
        int rs = k0 - c * g.RS;
        int r = rs / g.S;
        int s = rs - r * g.S;
#pragma unroll
        for (int i = 0; i < BK; ++i) {
            const int iy = iy0 + r * g.dh;
            const int ix = ix0 + s * g.dw;
            const bool ok = jvalid && (k0 + i < g.kdim) && (unsigned)iy < (unsigned)g.H &&
                            (unsigned)ix < (unsigned)g.W;
            v[i] = ok ? __ldg(xb + (int64_t)c * g.HW + iy * g.W + ix) : 0.f;
            if (++s == g.S) {
                s = 0;
                if (++r == g.R) {
                    r = 0;
                    ++c;
                }
            }
        }
    } else {
        const int64_t row0 = (p.pm.src_mode == SRC_MATRIX ? (int64_t)gi * g.kdim : 0) + k0;
        const float* base = p.src + lbase;
#pragma unroll
        for (int i = 0; i < BK; ++i) {
            const bool ok = jvalid && (k0 + i < g.kdim);
            v[i] = ok ? __ldg(base + (row0 + i) * lstride) : 0.f;
        }
    }
}

template <int BK, bool BF16>
__device__ __forceinline__ void store_split_row(uint8_t* a_hi, uint8_t* a_lo, int row,
                                                const float (&v)[BK]) {
    uint8_t* rh = a_hi + row * 128;
    uint8_t* rl = a_lo + row * 128;
    const int swz = row & 7;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const int off = ((q ^ swz) << 4);
        if (!BF16) {
            float4 h, l;
            Split2 s0 = split_tf32(v[4 * q + 0]);
            Split2 s1 = split_tf32(v[4 * q + 1]);
            Split2 s2 = split_tf32(v[4 * q + 2]);
            Split2 s3 = split_tf32(v[4 * q + 3]);
            h = make_float4(s0.hi, s1.hi, s2.hi, s3.hi);
            l = make_float4(s0.lo, s1.lo, s2.lo, s3.lo);
            *reinterpret_cast<float4*>(rh + off) = h;
            *reinterpret_cast<float4*>(rl + off) = l;
        } else {
            uint32_t h[4], l[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const float x0 = v[8 * q + 2 * e], x1 = v[8 * q + 2 * e + 1];
                const uint16_t h0 = bf16_rn_bits(x0), h1 = bf16_rn_bits(x1);
                const uint16_t l0 = bf16_rn_bits(x0 - bf16_bits_to_f32(h0));
                const uint16_t l1 = bf16_rn_bits(x1 - bf16_bits_to_f32(h1));
                h[e] = (uint32_t)h0 | ((uint32_t)h1 << 16);
                l[e] = (uint32_t)l0 | ((uint32_t)l1 << 16);
            }
            *reinterpret_cast<uint4*>(rh + off) = make_uint4(h[0], h[1], h[2], h[3]);
            *reinterpret_cast<uint4*>(rl + off) = make_uint4(l[0], l[1], l[2], l[3]);
        }
    }
}

template <int BN, int STAGES, bool BF16>
__global__ void __launch_bounds__(TC_THREADS, 1)
conv_tc_kernel(const __grid_constant__ TcParams p, const __grid_constant__ CUtensorMap tm_hi,
               const __grid_constant__ CUtensorMap tm_lo) {
    using Cfg = TcCfg<BN, STAGES, BF16>;
    constexpr int BK = Cfg::BK;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * Cfg::STAGE_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* tmem_full = empty + STAGES;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const Geom& g = p.g;
    const int tile_m = blockIdx.x;
    const int gi = blockIdx.y / p.n_tiles;
    const int tile_n = blockIdx.y - gi * p.n_tiles;
    const int kb_begin = blockIdx.z * p.kb_per_split;
    const int kb_end = min(p.num_kb, kb_begin + p.kb_per_split);
    const int nkb = kb_end - kb_begin;

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            ptx::mbar_init(&full[s], 128 + 1);
            ptx::mbar_init(&empty[s], 1);
        }
        ptx::mbar_init(tmem_full, 1);
        ptx::fence_mbar_init();
    }
    if (warp == 4 && lane == 0) {
        ptx::tma_prefetch_desc(&tm_hi);
        ptx::tma_prefetch_desc(&tm_lo);
    }
    if (warp == 5) ptx::tmem_alloc(tmem_slot, BN);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp < 4) {
        // ===================== activation producers, then epilogue =====================
        const int row = threadIdx.x;  // pixel row in the tile == TMEM lane
        const int64_t jl = (int64_t)tile_m * TC_BM + row;
        const bool jvalid = jl < p.pm.j_count;
        const int64_t j = p.pm.j_begin + jl;
        const float* xb = p.src;
        int iy0 = 0, ix0 = 0;
        int64_t lbase = 0, lstride = 0;
        if (p.pm.src_mode == SRC_CONV) {
            const int64_t jj = jvalid ? j : 0;
            const int64_t n = jj / g.PQ;
            const int pp = (int)(jj - n * g.PQ);
            const int oy = pp / g.Q;
            const int ox = pp - oy * g.Q;
            iy0 = oy * g.sh - g.ph;
            ix0 = ox * g.sw - g.pw;
            xb = p.src + (n * g.C + (int64_t)gi * g.cpg) * g.HW;
        } else if (jvalid) {
            src_linear(g, p.pm, j, lbase, lstride);
        }

        float v[BK];
        if (nkb > 0) gather_row<BK>(p, gi, kb_begin * BK, jvalid, xb, iy0, ix0, lbase, lstride, v);
        int stage = 0;
        uint32_t phase = 0;
        for (int i = 0; i < nkb; ++i) {
            ptx::mbar_wait(&empty[stage], phase ^ 1);
            uint8_t* st = smem + stage * Cfg::STAGE_BYTES;
            store_split_row<BK, BF16>(st, st + Cfg::A_BYTES, row, v);
            ptx::fence_proxy_async_smem();
            ptx::mbar_arrive(&full[stage]);
            if (i + 1 < nkb)
                gather_row<BK>(p, gi, (kb_begin + i + 1) * BK, jvalid, xb, iy0, ix0, lbase,
                               lstride, v);
            if (++stage == STAGES) {
                stage = 0;
                phase ^= 1;
            }
        }

        // ------------------------------- epilogue -------------------------------------
        ptx::mbar_wait(tmem_full, 0);
        ptx::tc_fence_after();
        int64_t obase = 0, ostride = 0;
        if (jvalid) dst_linear(g, p.pm, j, obase, ostride);
        const int f_tile0 = tile_n * BN;
#pragma unroll 1
        for (int c0 = 0; c0 < BN; c0 += 32) {
            if (f_tile0 + c0 >= g.kpg) break;  // warp-uniform
            uint32_t r[32];
            ptx::tmem_ld_32x32b_x32(tmem_base + ((uint32_t)(warp * 32) << 16) + c0, r);
            ptx::tmem_ld_wait();
            if (jvalid) {
#pragma unroll
                for (int i = 0; i < 32; ++i) {
                    const int fl = f_tile0 + c0 + i;
                    if (fl < g.kpg) {
                        const int f = gi * g.kpg + fl;
                        float* dst = p.out + obase + (int64_t)f * ostride;
                        const float a = __uint_as_float(r[i]);
                        if (p.add_mode)
                            atomicAdd(dst, a);
                        else
                            *dst = a + (p.bias ? __ldg(p.bias + f) : 0.f);
                    }
                }
            }
        }
    } else if (warp == 4) {
        // ============================ weight TMA producer =============================
        // converged warp, one elected lane issues (operands stay in uniform registers)
        const uint32_t leader = ptx::elect_one();
        const int row0 = gi * g.kpg + tile_n * BN;
        int stage = 0;
        uint32_t phase = 0;
        for (int i = 0; i < nkb; ++i) {
            ptx::mbar_wait(&empty[stage], phase ^ 1);
            uint8_t* st = smem + stage * Cfg::STAGE_BYTES;
            const int kc = (kb_begin + i) * BK;
            if (leader) {
                ptx::mbar_arrive_expect_tx(&full[stage], 2 * Cfg::B_BYTES);
                ptx::tma_load_2d(st + 2 * Cfg::A_BYTES, &tm_hi, &full[stage], kc, row0);
                ptx::tma_load_2d(st + 2 * Cfg::A_BYTES + Cfg::B_BYTES, &tm_lo, &full[stage], kc,
                                 row0);
            }
            __syncwarp();
            if (++stage == STAGES) {
                stage = 0;
                phase ^= 1;
            }
        }
    } else {
        // ============================== MMA issuer ====================================
        // converged warp; descriptors = stage-0 descriptors + constant offsets; one elected
        // lane issues
        constexpr uint32_t idesc = ptx::idesc_f32acc<BF16>(TC_BM, BN);
        constexpr uint32_t STG16 = Cfg::STAGE_BYTES >> 4;
        constexpr uint32_t ALO16 = Cfg::A_BYTES >> 4, BLO16 = Cfg::B_BYTES >> 4;
        const uint32_t s0 = ptx::smem_u32(smem);
        const uint64_t da0 = ptx::sdesc_k_sw128(s0);
        const uint64_t db0 = ptx::sdesc_k_sw128(s0 + 2 * Cfg::A_BYTES);
        const uint32_t leader = ptx::elect_one();
        int stage = 0;
        uint32_t phase = 0;
        for (int i = 0; i < nkb; ++i) {
            ptx::mbar_wait(&full[stage], phase);
            ptx::tc_fence_after();
            const uint64_t sa = da0 + (uint64_t)(stage * STG16);
            const uint64_t sb = db0 + (uint64_t)(stage * STG16);
            if (leader) {
#pragma unroll
                for (int kk = 0; kk < BK / Cfg::UK; ++kk) {
                    const uint64_t dah = sa + 2 * kk;  // 32 bytes along the swizzled row
                    const uint64_t dal = dah + ALO16;
                    const uint64_t dbh = sb + 2 * kk;
                    const uint64_t dbl = dbh + BLO16;
                    // small terms first, then the dominant hi*hi product
                    ptx::umma<BF16>(tmem_base, dal, dbh, idesc, (i | kk) != 0);
                    ptx::umma<BF16>(tmem_base, dah, dbl, idesc, 1);
                    ptx::umma<BF16>(tmem_base, dah, dbh, idesc, 1);
                }
                ptx::umma_commit(&empty[stage]);
            }
            __syncwarp();
            if (++stage == STAGES) {
                stage = 0;
                phase ^= 1;
            }
        }
        if (leader) ptx::umma_commit(tmem_full);
        __syncwarp();
    }

    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 5) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem_base, BN);
    }
}

// ----------------------------------------------------------------------------------------
// Host side
// ----------------------------------------------------------------------------------------
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
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

static int make_wmap(CUtensorMap* m, bool bf16, const void* w, int rows, int kdim_pad, int bk,
                     int bn) {
    auto fn = encode_fn();
    if (!fn) return fail(CB_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    if (reinterpret_cast<uintptr_t>(w) & 15)
        return fail(CB_ERR_MISALIGNED, "split weights must be 16-byte aligned");
    const int eb = bf16 ? 2 : 4;
    cuuint64_t dims[2] = {(cuuint64_t)kdim_pad, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)kdim_pad * eb};
    cuuint32_t box[2] = {(cuuint32_t)bk, (cuuint32_t)bn};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(m, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                    const_cast<void*>(w), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(CB_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
    return CB_OK;
}

template <int BN, int STAGES, bool BF16>
static int launch_cfg(const TcParams& prm, dim3 grid, const void* w_hi, const void* w_lo,
                      cudaStream_t st) {
    using Cfg = TcCfg<BN, STAGES, BF16>;
    static std::once_flag once;
    static cudaError_t attr_err = cudaSuccess;
    std::call_once(once, [] {
        attr_err = cudaFuncSetAttribute(conv_tc_kernel<BN, STAGES, BF16>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        Cfg::SMEM_BYTES);
    });
    if (attr_err != cudaSuccess)
        return fail(CB_ERR_CUDA, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(attr_err));
    CUtensorMap mh, ml;
    const int rows = prm.g.G * prm.g.kpg;
    int rc = make_wmap(&mh, BF16, w_hi, rows, prm.g.kdim_pad, Cfg::BK, BN);
    if (rc) return rc;
    rc = make_wmap(&ml, BF16, w_lo, rows, prm.g.kdim_pad, Cfg::BK, BN);
    if (rc) return rc;
    conv_tc_kernel<BN, STAGES, BF16><<<grid, TC_THREADS, Cfg::SMEM_BYTES, st>>>(prm, mh, ml);
    return check_launch("conv_tc_kernel");
}

struct TcPlan {
    int bn, stages, splits, kb_per_split, num_kb, n_tiles;
    int64_t m_tiles;
};

// Tile/split heuristic: fill the 148 SMs, prefer wide N tiles (fewer activation
// re-gathers), split K when the M x N grid cannot fill the machine.
static TcPlan plan_tc(const Geom& g, int64_t npix, bool bf16, bool allow_split) {
    TcPlan pl{};
    const int bk = bf16 ? 64 : 32;
    pl.num_kb = (g.kdim + bk - 1) / bk;
    pl.m_tiles = ceil_div64(npix, TC_BM);
    const int sms = sm_count();
    int best_bn = 64;
    double best_cost = 1e300;
    for (int bn : {256, 128, 64}) {
        if (bn > 64 && g.kpg <= bn / 2) continue;  // mostly-empty tile
        const int64_t tiles = pl.m_tiles * ((g.kpg + bn - 1) / bn) * g.G;
        const double waves = std::ceil((double)tiles / sms);
        // per-tile cost ~ MMA cycles (bn * num_kb) + fixed gather/epilogue overhead
        const double cost = waves * ((double)bn * pl.num_kb + 64.0 * 40 + bn * 8.0);
        if (cost < best_cost * 0.97) {
            best_cost = cost;
            best_bn = bn;
        }
    }
    pl.bn = best_bn;
    pl.n_tiles = (g.kpg + pl.bn - 1) / pl.bn;
    const int64_t tiles = pl.m_tiles * pl.n_tiles * g.G;
    pl.splits = 1;
    if (allow_split && tiles < sms && pl.num_kb >= 4) {
        int want = (int)((sms + tiles - 1) / tiles);
        want = std::min(want, pl.num_kb / 2);
        pl.splits = std::max(1, want);
    }
    // accumulator promotion (promote_k): no CTA accumulates more than ~promote_k reduction
    // elements; the K splits are added into the pre-initialised output in fp32
    if (allow_split) pl.splits = std::max(pl.splits, (pl.num_kb * bk + promote_k(bf16) - 1) / promote_k(bf16));
    pl.kb_per_split = (pl.num_kb + pl.splits - 1) / pl.splits;
    pl.splits = (pl.num_kb + pl.kb_per_split - 1) / pl.kb_per_split;
    const int kb_cta = pl.kb_per_split;
    if (pl.bn == 256) pl.stages = 2;
    else if (pl.bn == 128) pl.stages = kb_cta <= 3 ? 2 : 3;
    else pl.stages = kb_cta <= 3 ? 2 : 4;
    return pl;
}

// Launches the tensor-core kernel.  add_mode: 0 store (+bias), 1 accumulate into out.
// When the plan splits K and add_mode==0 the output is first initialised (bias or zero)
// and the splits accumulate into it.

int tc_plan_query(const Geom& g, int64_t npix, bool bf16, bool allow_split, cb_tile_plan* out) {
    TcPlan pl = plan_tc(g, npix, bf16, allow_split);
    out->variant = bf16 ? CB_VARIANT_TC3XBF16 : CB_VARIANT_TC3XTF32;
    out->block_m = TC_BM;
    out->block_n = pl.bn;
    out->block_k = bf16 ? 64 : 32;
    out->stages = pl.stages;
    out->splits = pl.splits;
    out->m_tiles = pl.m_tiles;
    out->n_tiles = (int64_t)pl.n_tiles * g.G;
    out->k_blocks = pl.num_kb;
    out->ctas = pl.m_tiles * pl.n_tiles * g.G * pl.splits;
    return CB_OK;
}

// zero_kind: how a split-K output can be pre-initialised when add_mode == 0:
//   0 = it cannot (never split), 1 = NCHW bias fill, 2 = contiguous K*npix memset.
int pre_init_output(const Geom& g, const PixMap& pm, int zero_kind, const float* bias, float* out,
                    cudaStream_t st);

int launch_tc(bool bf16, const Geom& g, const PixMap& pm, const float* src, const void* w_hi,
              const void* w_lo, const float* bias, float* out, int add_mode, int zero_kind,
              cudaStream_t st) {
    if (pm.j_count == 0) return CB_OK;
    TcPlan pl = plan_tc(g, pm.j_count, bf16, add_mode || zero_kind != 0);
    TcParams prm{};
    prm.g = g;
    prm.pm = pm;
    prm.src = src;
    prm.bias = bias;
    prm.out = out;
    prm.num_kb = pl.num_kb;
    prm.kb_per_split = pl.kb_per_split;
    prm.n_tiles = pl.n_tiles;
    prm.add_mode = add_mode;
    if (pl.splits > 1 && !add_mode) {
        int rc = pre_init_output(g, pm, zero_kind, bias, out, st);
        if (rc) return rc;
        prm.add_mode = 1;
    }
    if (pl.m_tiles > 0x7fffffffLL) return fail(CB_ERR_UNSUPPORTED, "too many pixel tiles");
    dim3 grid((unsigned)pl.m_tiles, (unsigned)(pl.n_tiles * g.G), (unsigned)pl.splits);
#define CB_TC_CASE(BN_, ST_)                                                              \
    if (pl.bn == BN_ && pl.stages == ST_)                                                 \
        return bf16 ? launch_cfg<BN_, ST_, true>(prm, grid, w_hi, w_lo, st)               \
                    : launch_cfg<BN_, ST_, false>(prm, grid, w_hi, w_lo, st);
    CB_TC_CASE(256, 2)
    CB_TC_CASE(128, 3)
    CB_TC_CASE(128, 2)
    CB_TC_CASE(64, 4)
    CB_TC_CASE(64, 2)
#undef CB_TC_CASE
    return fail(CB_ERR_UNSUPPORTED, "no tensor-core tile configuration");
}

}  // namespace cb
