// conv_gemm_ts.cu -- K8: the stepwise algorithms' GEMM microkernel (im2col matrix or SConv
// slice buffer x split weights) on tcgen05 with the A operand built in TMEM.
//
// K4 (conv_tc.cu) gathers its fp32 operand per thread into a swizzled smem tile, one tile
// per CTA (not persistent, wave-quantized).  K8 instead:
//
//   * warps 0-7 (producers, two per TMEM lane quadrant, alternating 32-wide K chunks) read
//     the fp32 operand rows -- pixel j, reduction k at base(j) + k*stride(j), coalesced along
//     pixels -- split each value (bf16 or tf32 hi/lo) and write the chunk straight into a
//     TMEM ring with tcgen05.st;
//   * warp 12 TMA-streams the split weight tiles (K-major, SWIZZLE_128B) through an smem ring;
//   * warp 13 issues A_lo*B_hi, A_hi*B_lo, A_hi*B_hi per K step with A read from TMEM;
//   * warps 8-11 drain the accumulator through the PixMap output modes (NCHW + bias, SConv
//     slice accumulators, or a row-major matrix, optionally accumulating into it).
//
// Persistent: one CTA per SM walks (pixel tile, channel tile, group) items.
#include <cudaTypedefs.h>

#include <mutex>

#include "cb_common.cuh"
#include "sm100_ptx.cuh"

namespace cb {

unsigned long long* debug_trace_buffer(int ctas, cudaStream_t st);  // conv_tma.cu

constexpr int G8_BM = 128;
constexpr int G8_PROD_WARPS = 8;
constexpr int G8_EPI_WARP0 = 8;   // warps 8-15: two epilogue warps per TMEM lane quadrant
constexpr int G8_EPI_THREADS = 256;
constexpr int G8_TMA_WARP = 16;
constexpr int G8_MMA_WARP = 17;
constexpr int G8_ATMA_WARP = 18;  // A tiles by TMA (matrix sources)
constexpr int G8_THREADS = 19 * 32;
constexpr int G8_ASTAGES_MAX = 8;
constexpr int G8_ASTAGE_BYTES = 32 * G8_BM * 4;  // [32 k][128 px] fp32
constexpr int G8_TMEM_COLS = 512;
constexpr int G8_CK = 32;  // reduction elements per A chunk
constexpr int G8_OSTAGE_BYTES = 32 * 32 * 4;  // per epilogue warp: [32 channels][32 pixels] fp32

struct G8Params {
    Geom g;
    PixMap pm;
    const float* src;
    const float* bias;
    float* out;
    int add_mode;     // 1: out += acc (no bias), 0: out = acc (+bias)
    int n_tiles;      // channel tiles per group
    int64_t m_tiles;  // pixel tiles
    int64_t items;    // m_tiles * n_tiles * G
    int nchunks;      // ceil(kdim / 32)
    int ring;         // A chunks in the TMEM ring
    int bstages;      // smem weight stages
    int tma_a;        // 1: A chunks arrive by TMA into smem, 0: per-thread loads
    // Tail N-split: items [0, full_items) are whole tiles; each of the remaining tiles (the
    // ragged last wave) is cut into tail_split channel ranges (multiples of 16 columns), one
    // item each, so the last wave keeps every SM busy.  A is rebuilt per range.
    int64_t full_items;
    int tail_split;
    // Tail K-split (tail_k = 1, instead of the N split): each tail tile is cut into
    // tail_split balanced ranges of its reduction chunks, one item each (full N, A built once
    // per chunk overall).  The parts run concurrently in the last wave (one per CTA) and add
    // into y in part order: the warp of lane quadrant q for column chunk c of part p > 0
    // waits until flags[(tau * col_chunks + c) * 4 + q] == p, adds, and hands on p + 1 (the
    // last part resets it to 0) -- deterministic, no workspace.
    int tail_k;
    uint32_t* flags;
    // Accumulator promotion: the tensor core's fp32 accumulation truncates, so its error
    // grows faster than linearly with the number of MMAs into one accumulator (measured on
    // the config-5 sweep: up to 1.3e-3 normalized at C*R*S = 100352).  Every range_chunks
    // chunks (of 32 reduction elements) the accumulator is drained by the epilogue and
    // added to the output in fp32 (round to nearest), then restarted.
    int range_chunks;
    unsigned long long* trace;  // diagnostics (CB_K8_TRACE): per-CTA globaltimer stamps
    int astages;                // A chunk stages in smem (TMA sources)
    int debug;                  // diagnostics (CB_K8_DEBUG): 1 no weight TMA, 2 no A TMA, 4 no MMA, 8 no A build, 16 no epilogue stores, 32 no bias
    // TMA-store epilogue (tma_y = 1: NCHW y as {PQ, K, N}; 2: a row-major output matrix as
    // {ld, rows, 1}, e.g. the SConv accumulators): an epilogue warp stages its 32 rows x 32
    // channels in smem and one lane stores them with the TMA engine; warps whose rows cross
    // an image or hold invalid rows and partial channel chunks use per-lane stores
    int tma_y;
};

__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t* f) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_gpu(uint32_t* f, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(f), "r"(v) : "memory");
}

// Hand-off flags of the K-split tail (G8Params::tail_k), a static pool: every launch takes
// the next free run of slots (host side, round robin) and leaves them at 0.  Two K8 launches
// running at the same time only share slots after 64K slots of other launches.
constexpr int G8_FLAG_SLOTS = 1 << 16;
__device__ uint32_t g8_flags[G8_FLAG_SLOTS];

// CB_K8_TRACE chunk stamps of CTA 0 (chunk cg < 256): [8192 + 4 cg + e], e: 0 A TMA
// issued, 1 producer group saw the A stage, 2 producer arrived a_full, 3 MMA saw a_full
__device__ __forceinline__ void g8_cstamp(const struct G8Params& p, int64_t cg, int e);
// CB_K8_TRACE stamps, [cta][32]: slot li*6 + e for the CTA's local item li < 5 (e: 0/1
// producer warp 0 starts / finishes the item, 2/3 MMA first chunk issued / last commit,
// 4/5 epilogue accumulator ready / last store issued), 30 kernel end, 31 kernel start
__device__ __forceinline__ void g8_stamp(const G8Params& p, int slot) {
    if (kTrace && p.trace && slot < 32) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        p.trace[blockIdx.x * 32 + slot] = t;
    }
}
__device__ __forceinline__ void g8_cstamp(const G8Params& p, int64_t cg, int e) {
    if (kTrace && p.trace && blockIdx.x == 0 && cg < 256) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        p.trace[8192 + 4 * cg + e] = t;
    }
}

// channel range [lo, hi) of part `sub` of a BN-wide tile cut into `parts` (16-aligned)
__device__ __forceinline__ int g8_part_col(int bn, int parts, int sub) {
    return min(bn, ((bn * sub / parts) + 15) / 16 * 16);
}

template <int BN, bool BF16>
struct G8Cfg {
    static constexpr int EB = BF16 ? 2 : 4;
    static constexpr int KE = 128 / EB;            // reduction per weight stage (128-byte rows)
    static constexpr int CPS = KE / G8_CK;         // A chunks per weight stage: 2 (bf16), 1 (tf32)
    static constexpr int UK = 32 / EB;             // reduction per MMA
    static constexpr int HALF_COLS = G8_CK * EB / 4;  // TMEM columns of one half of a chunk
    static constexpr int CHUNK_COLS = 2 * HALF_COLS;
    static constexpr int B_BYTES = BN * 128;       // one half (hi or lo) of a weight stage
    static constexpr int STAGE_BYTES = 2 * B_BYTES;
};

template <int BN, bool BF16>
__global__ void __launch_bounds__(G8_THREADS, 1)
gemm_ts_kernel(const __grid_constant__ G8Params p, const __grid_constant__ CUtensorMap tm_hi,
               const __grid_constant__ CUtensorMap tm_lo, const __grid_constant__ CUtensorMap tm_a,
               const __grid_constant__ CUtensorMap tm_y) {
    using Cfg = G8Cfg<BN, BF16>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    float* astage = reinterpret_cast<float*>(smem + p.bstages * Cfg::STAGE_BYTES);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + p.bstages * Cfg::STAGE_BYTES +
                                                 p.astages * G8_ASTAGE_BYTES);
    uint64_t* b_full = bars;                    // [bstages]
    uint64_t* b_empty = b_full + p.bstages;     // [bstages]
    uint64_t* a_full = b_empty + p.bstages;     // [ring]
    uint64_t* a_empty = a_full + p.ring;        // [ring]
    uint64_t* acc_full = a_empty + p.ring;      // 1
    uint64_t* acc_empty = acc_full + 1;         // 1
    uint64_t* as_full = acc_empty + 1;          // [astages]
    uint64_t* as_empty = as_full + p.astages;   // [astages]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(as_empty + p.astages);
    // epilogue staging, one 4 KB buffer per epilogue warp (1 KB after the barriers)
    float* ostage = reinterpret_cast<float*>(smem + p.bstages * Cfg::STAGE_BYTES +
                                             p.astages * G8_ASTAGE_BYTES + 1024);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const Geom& g = p.g;

    if (threadIdx.x == 0) {
        for (int s = 0; s < p.bstages; ++s) {
            ptx::mbar_init(&b_full[s], 1);
            ptx::mbar_init(&b_empty[s], 1);
        }
        for (int s = 0; s < p.ring; ++s) {
            ptx::mbar_init(&a_full[s], 128);
            ptx::mbar_init(&a_empty[s], 1);
        }
        ptx::mbar_init(acc_full, 1);
        ptx::mbar_init(acc_empty, G8_EPI_THREADS);
        for (int s = 0; s < p.astages; ++s) {
            ptx::mbar_init(&as_full[s], 1);
            ptx::mbar_init(&as_empty[s], 128);
        }
        ptx::fence_mbar_init();
    }
    if (warp == G8_TMA_WARP && lane == 0) {
        ptx::tma_prefetch_desc(&tm_hi);
        ptx::tma_prefetch_desc(&tm_lo);
    }
    if (warp == G8_MMA_WARP) ptx::tmem_alloc(tmem_slot, G8_TMEM_COLS);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const int nch = p.nchunks;
    if (threadIdx.x == 0) g8_stamp(p, 31);

    // pixel tile mt, row m -> launch-local pixel jl
    auto pix_of = [&](int64_t mt, int m, int64_t& jl) -> bool {
        jl = mt * G8_BM + m;
        return jl < p.pm.j_count;
    };
    // item -> (channel tile nt, pixel tile mt, group gi; tile columns [c_lo, c_hi))
    // K-split tail parts: reduction chunks [k_lo, k_hi), part index and tail tile tau
    int c_lo = 0, c_hi = BN, k_lo = 0, k_hi = nch, kpart = -1, ktau = 0;
    auto decode = [&](int64_t t, int& nt, int64_t& mt, int& gi) {
        c_lo = 0;
        c_hi = BN;
        k_lo = 0;
        k_hi = nch;
        kpart = -1;
        if (t >= p.full_items) {
            const int64_t j = t - p.full_items;
            const int sub = (int)(j % p.tail_split);
            t = p.full_items + j / p.tail_split;
            if (p.tail_k) {
                kpart = sub;
                ktau = (int)(j / p.tail_split);
                k_lo = nch * sub / p.tail_split;
                k_hi = nch * (sub + 1) / p.tail_split;
            } else {
                c_lo = g8_part_col(BN, p.tail_split, sub);
                c_hi = g8_part_col(BN, p.tail_split, sub + 1);
            }
        }
        nt = (int)(t % p.n_tiles);
        const int64_t r = t / p.n_tiles;
        mt = r % p.m_tiles;
        gi = (int)(r / p.m_tiles);
    };

    if (warp < G8_PROD_WARPS) {
        // ============================ A producers ======================================
        const int quad = warp & 3, kpar = warp >> 2;
        const int m = quad * 32 + lane;
        const uint32_t lane_tm = tmem_base + ((uint32_t)(quad * 32) << 16) + BN;  // ring base
        int64_t cbase = 0;  // chunks this CTA produced before the current item
        int li = 0;
        // This group's next global chunk cg (cg == kpar mod 2) and its TMEM ring slot / A
        // stage with their phases, advanced incrementally: per-chunk 64-bit div/mod by the
        // runtime ring and stage counts had cost ~1300 cycles a chunk on the MMA's critical
        // path (K8's MMAs ran at ~45% of the tcgen05 rate with every operand disabled).
        int64_t cg = kpar;
        int slot = kpar % p.ring, as = kpar;  // astages is even (>= 2)
        uint32_t ph = (uint32_t)(kpar / p.ring), asph = 0;
        auto advance = [&] {
            cg += 2;
            if ((slot += 2) >= p.ring) {
                slot -= p.ring;
                ph ^= 1;
            }
            if ((as += 2) >= p.astages) {
                as -= p.astages;
                asph ^= 1;
            }
        };
        for (int64_t t = blockIdx.x; t < p.items; t += gridDim.x, cbase += k_hi - k_lo, ++li) {
            int nt, gi;
            int64_t mt;
            decode(t, nt, mt, gi);
            if (threadIdx.x == 0 && li < 5) g8_stamp(p, li * 6);
            int64_t jl;
            const bool jvalid = pix_of(mt, m, jl);
            int64_t lbase = 0, lstride = 0;
            if (jvalid) src_linear(g, p.pm, p.pm.j_begin + jl, lbase, lstride);
            const int64_t row0 = p.pm.src_mode == SRC_MATRIX ? (int64_t)gi * g.kdim : 0;
            const float* srcp = p.src + lbase + row0 * lstride;
            // chunks go to producer groups by GLOBAL chunk parity (cg & 1): each A stage
            // (cg % 4) is then always consumed by the same group, so its phase parity can never
            // alias an older phase (with kc parity, an odd chunk count per item would hand a
            // stage to the other group on the next item -- an ABA race on the mbarrier phase)
            for (int kc = k_lo + (int)(cg - cbase); kc < k_hi; kc += 2) {
                float v[G8_CK];
                const int k0 = kc * G8_CK;
                if (p.tma_a) {  // the chunk's [32 k][128 px] box is in smem: read column m
                    ptx::mbar_wait(&as_full[as], asph);
                    if (lane == 0 && quad == 0) g8_cstamp(p, cg, 1);
                    const float* col = astage + (size_t)as * (32 * G8_BM) + m;
                    if (p.debug & 8) {  // diagnostics: no A build (stale TMEM A)
                        ptx::mbar_arrive(&as_empty[as]);
                        ptx::mbar_wait(&a_empty[slot], ph ^ 1);
                        ptx::tc_fence_before();
                        ptx::mbar_arrive(&a_full[slot]);
                        advance();
                        continue;
                    }
#pragma unroll
                    for (int e = 0; e < G8_CK; ++e) v[e] = col[e * G8_BM];
                    ptx::mbar_arrive(&as_empty[as]);
                } else {
#pragma unroll
                    for (int e = 0; e < G8_CK; ++e)
                        v[e] = (jvalid && k0 + e < g.kdim) ? __ldg(srcp + (int64_t)(k0 + e) * lstride) : 0.f;
                }
                ptx::mbar_wait(&a_empty[slot], ph ^ 1);
                ptx::tc_fence_after();
                const uint32_t a_hi = lane_tm + slot * Cfg::CHUNK_COLS;
                const uint32_t a_lo = a_hi + Cfg::HALF_COLS;
                if (BF16) {
                    uint32_t hv[16], lv[16];
#pragma unroll
                    for (int e = 0; e < 16; ++e) {  // paired conversions (2 values per cvt)
                        const float a0 = v[2 * e], a1 = v[2 * e + 1];
                        uint32_t h;
                        asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(h) : "f"(a1), "f"(a0));
                        const float r0 = a0 - __uint_as_float(h << 16), r1 = a1 - __uint_as_float(h & 0xffff0000u);
                        uint32_t l;
                        asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(l) : "f"(r1), "f"(r0));
                        hv[e] = h;
                        lv[e] = l;
                    }
                    ptx::tmem_st_32x32b_x16(a_hi, hv);
                    ptx::tmem_st_32x32b_x16(a_lo, lv);
                } else {
                    uint32_t hv[32], lv[32];
#pragma unroll
                    for (int e = 0; e < 32; ++e) {
                        const Split2 sp = split_tf32(v[e]);
                        hv[e] = __float_as_uint(sp.hi);
                        lv[e] = __float_as_uint(sp.lo);
                    }
                    ptx::tmem_st_32x32b_x32(a_hi, hv);
                    ptx::tmem_st_32x32b_x32(a_lo, lv);
                }
                ptx::tmem_st_wait();
                ptx::tc_fence_before();
                ptx::mbar_arrive(&a_full[slot]);
                if (lane == 0 && quad == 0) g8_cstamp(p, cg, 2);
                advance();
            }
            if (threadIdx.x == 0 && li < 5) g8_stamp(p, li * 6 + 1);
        }
    } else if (warp < G8_TMA_WARP) {
        // ============================ epilogue ==========================================
        // Two warps per lane quadrant, alternating 32-column chunks: the single accumulator
        // is released only once it is fully read, and each warp's reads wait behind its own
        // stores, so a second warp halves the time the MMAs of the next item wait for it.
        const int quad = warp & 3, ehalf = (warp - G8_EPI_WARP0) >> 2;
        const int m = quad * 32 + lane;
        int i = 0;  // accumulator ranges drained so far (acc_full phase)
        int li = 0;
        for (int64_t t = blockIdx.x; t < p.items; t += gridDim.x, ++li) {
            int nt, gi;
            int64_t mt;
            decode(t, nt, mt, gi);
            int64_t jl;
            const bool jvalid = pix_of(mt, m, jl);
            int64_t obase = 0, ostride = 0;
            if (jvalid) dst_linear(g, p.pm, p.pm.j_begin + jl, obase, ostride);
            const int f_tile0 = nt * BN + c_lo;
            const int ncol = min(c_hi - c_lo, g.kpg - f_tile0);
            const int nranges = (k_hi - k_lo + p.range_chunks - 1) / p.range_chunks;
            const bool kord = kpart >= 0;  // K-split tail part (one range): ordered adds
#pragma unroll 1
            for (int rg = 0; rg < nranges; ++rg, ++i) {
            ptx::mbar_wait(acc_full, i & 1);
            ptx::tc_fence_after();
            if (threadIdx.x == G8_EPI_WARP0 * 32 && rg == 0 && li < 5) g8_stamp(p, li * 6 + 4);
            if (32 * ehalf >= ncol) {  // no column chunk for this warp: release at once
                ptx::tc_fence_before();
                ptx::mbar_arrive(acc_empty);
            }
            // later ranges, and later K parts, add to what is already stored
            const bool add = p.add_mode || rg > 0 || kpart > 0;
#pragma unroll 1
            for (int c0 = 32 * ehalf; c0 < ncol; c0 += 64) {
                uint32_t r[32];
                ptx::tmem_ld_32x32b_x32(tmem_base + ((uint32_t)(quad * 32) << 16) + c0, r);
                ptx::tmem_ld_wait();
                if (c0 + 64 >= ncol) {  // this warp's part of the accumulator is read
                    ptx::tc_fence_before();
                    ptx::mbar_arrive(acc_empty);
                }
                uint32_t* flag = kord ? p.flags + ((size_t)(ktau * (BN / 32) + c0 / 32) * 4 + quad) : nullptr;
                if (kord && kpart > 0) {  // the previous part's rows of this chunk are stored
                    if (lane == 0) {
                        while (ld_acquire_gpu(flag) != (uint32_t)kpart) __nanosleep(64);
                        asm volatile("fence.proxy.async.global;" ::: "memory");  // before a TMA add
                    }
                    __syncwarp();
                }
                const int nvalid = min(32, ncol - c0);
                const int fb = gi * g.kpg + f_tile0 + c0;
                // TMA store (or TMA add for later ranges / K parts / add_mode) of this warp's
                // 32 x 32 block: every row valid and in one image (NCHW), a whole channel
                // chunk
                bool tma_ok = p.tma_y && nvalid == 32 && !(p.debug & 16) && __all_sync(0xffffffffu, jvalid);
                int32_t yc0 = 0, yc2 = 0;
                if (tma_ok) {
                    const int64_t ja = p.pm.j_begin + jl;
                    if (p.tma_y == 1) {
                        const int64_t n = ja / g.PQ;
                        yc0 = (int32_t)(ja - n * g.PQ);
                        yc2 = (int32_t)n;
                    } else {  // output matrix: column ja
                        yc0 = (int32_t)ja;
                    }
                    const int32_t y2_0 = __shfl_sync(0xffffffffu, yc2, 0);
                    tma_ok = __all_sync(0xffffffffu, y2_0 == yc2);  // one image
                    yc0 = __shfl_sync(0xffffffffu, yc0, 0);
                    yc2 = y2_0;
                }
                if (tma_ok) {
                    float* buf = ostage + (warp - G8_EPI_WARP0) * (G8_OSTAGE_BYTES / 4);
                    if (lane == 0) ptx::bulk_wait_read<0>();  // this warp's previous store left buf
                    __syncwarp();
#pragma unroll
                    for (int e = 0; e < 32; ++e)
                        buf[e * 32 + lane] = __uint_as_float(r[e]) +
                                             (!add && p.bias && !(p.debug & 32) ? __ldg(p.bias + fb + e) : 0.f);
                    ptx::fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) {
                        if (add) {
                            // a later range of this CTA adds onto its own earlier store of the
                            // chunk: make sure that store has landed
                            if (!kord) ptx::bulk_wait_all();
                            ptx::tma_reduce_add_3d(&tm_y, buf, yc0, fb, yc2);
                        } else {
                            ptx::tma_store_3d(&tm_y, buf, yc0, fb, yc2);
                        }
                        ptx::bulk_commit();
                    }
                } else if (jvalid && !(p.debug & 16)) {
                float* dst = p.out + obase + (int64_t)fb * ostride;
                if (add) {  // all loads of a half before its first store (no per-element round trips)
#pragma unroll
                    for (int h = 0; h < 32; h += 16) {
                        float o[16];
#pragma unroll
                        for (int e = 0; e < 16; ++e)
                            o[e] = h + e < nvalid ? __ldcg(dst + (int64_t)(h + e) * ostride) : 0.f;
#pragma unroll
                        for (int e = 0; e < 16; ++e)
                            if (h + e < nvalid) dst[(int64_t)(h + e) * ostride] = __uint_as_float(r[h + e]) + o[e];
                    }
                } else {
#pragma unroll
                    for (int e = 0; e < 32; ++e)
                        if (e < nvalid)
                            dst[(int64_t)e * ostride] =
                                __uint_as_float(r[e]) + (p.bias && !(p.debug & 32) ? __ldg(p.bias + fb + e) : 0.f);
                }
                }
                if (kord) {  // hand the chunk on to the next part (the last one resets the flag)
                    if (tma_ok && lane == 0) {  // the TMA store / add has landed in global memory
                        ptx::bulk_wait_all();
                        asm volatile("fence.proxy.async.global;" ::: "memory");
                    }
                    __threadfence();
                    __syncwarp();
                    if (lane == 0) st_release_gpu(flag, kpart + 1 == p.tail_split ? 0u : (uint32_t)(kpart + 1));
                }
            }
            }
            if (threadIdx.x == G8_EPI_WARP0 * 32 && li < 5) g8_stamp(p, li * 6 + 5);
        }
        if (lane == 0 && p.tma_y) ptx::bulk_wait_all();
    } else if (warp == G8_ATMA_WARP) {
        // ============================ A chunks by TMA (matrix sources) ==================
        if (p.tma_a) {
            const uint32_t leader = ptx::elect_one();
            int64_t cbase = 0;
            int as = 0;
            uint32_t asph = 0;
            for (int64_t t = blockIdx.x; t < p.items; t += gridDim.x, cbase += k_hi - k_lo) {
                int nt, gi;
                int64_t mt;
                decode(t, nt, mt, gi);
                const int x0 = (int)(p.pm.j_begin + mt * G8_BM);
                const int row0 = gi * g.kdim;
                for (int kc = k_lo; kc < k_hi; ++kc, as = as + 1 == p.astages ? 0 : as + 1,
                         asph ^= (as == 0 ? 1u : 0u)) {
                    const int64_t cg = cbase + (kc - k_lo);
                    ptx::mbar_wait(&as_empty[as], asph ^ 1);
                    if (leader) g8_cstamp(p, cg, 0);
                    if (leader && (p.debug & 2) && cg >= p.astages) {
                        ptx::mbar_arrive(&as_full[as]);  // diagnostics: stale A chunk
                    } else if (leader) {
                        ptx::mbar_arrive_expect_tx(&as_full[as], G8_ASTAGE_BYTES);
                        ptx::tma_load_2d(astage + (size_t)as * (32 * G8_BM), &tm_a, &as_full[as], x0,
                                             row0 + kc * G8_CK);
                    }
                    __syncwarp();
                }
            }
        }
    } else if (warp == G8_TMA_WARP) {
        // ============================ weight TMA =========================================
        const uint32_t leader = ptx::elect_one();
        int64_t sbase = 0;
        int s = 0;
        uint32_t ph = 0;
        for (int64_t t = blockIdx.x; t < p.items; t += gridDim.x) {
            int nt, gi;
            int64_t mt;
            decode(t, nt, mt, gi);
            const int nstage = (k_hi - k_lo + Cfg::CPS - 1) / Cfg::CPS;
            const int row0 = gi * g.kpg + nt * BN + c_lo;  // (a part's rows start the stage)
            for (int kb = 0; kb < nstage; ++kb, s = s + 1 == p.bstages ? 0 : s + 1, ph ^= (s == 0 ? 1u : 0u)) {
                const int64_t sg = sbase + kb;
                ptx::mbar_wait(&b_empty[s], ph ^ 1);
                if (leader && (p.debug & 1) && sg >= p.bstages) {
                    ptx::mbar_arrive(&b_full[s]);  // diagnostics: stale weights, no transfer
                } else if (leader) {
                    uint8_t* st = smem + s * Cfg::STAGE_BYTES;
                    ptx::mbar_arrive_expect_tx(&b_full[s], Cfg::STAGE_BYTES);
                    const int kx = k_lo * G8_CK + kb * Cfg::KE;
                    ptx::tma_load_2d(st, &tm_hi, &b_full[s], kx, row0);
                    ptx::tma_load_2d(st + Cfg::B_BYTES, &tm_lo, &b_full[s], kx, row0);
                }
                __syncwarp();
            }
        }
    } else {
        // ============================ MMA issuer ========================================
        const uint32_t leader = ptx::elect_one();
        constexpr uint32_t idesc_full = ptx::idesc_f32acc<BF16>(G8_BM, BN);
        const uint64_t db0 = ptx::sdesc_k_sw128(ptx::smem_u32(smem));
        constexpr uint32_t STG16 = Cfg::STAGE_BYTES >> 4, BLO16 = Cfg::B_BYTES >> 4;
        int64_t cbase = 0;
        int slot = 0, s = 0;  // TMEM A ring slot and weight stage, with their phases
        uint32_t aph = 0, bph = 0;
        int i = 0;  // accumulator ranges issued so far (acc_empty phase)
        int li = 0;
        for (int64_t t = blockIdx.x; t < p.items; t += gridDim.x, cbase += k_hi - k_lo, ++li) {
            int nt, gi;
            int64_t mt;
            decode(t, nt, mt, gi);
            const uint32_t idesc =
                c_hi - c_lo == BN ? idesc_full : ptx::idesc_f32acc<BF16>(G8_BM, c_hi - c_lo);
            int kr = 0;  // position inside the accumulator range
            for (int kc = k_lo; kc < k_hi; ++kc) {
                const int j = kc - k_lo;  // chunk of this item (weight stages start at k_lo)
                if (kr == 0) {  // a fresh accumulator range: the epilogue drained the last one
                    if (j > 0) {
                        if (leader) ptx::umma_commit(acc_full);
                        __syncwarp();
                        ++i;
                    }
                    ptx::mbar_wait(acc_empty, (i & 1) ^ 1);
                    ptx::tc_fence_after();
                }
                const int64_t cg = cbase + j;
                if (j % Cfg::CPS == 0) ptx::mbar_wait(&b_full[s], bph);
                ptx::mbar_wait(&a_full[slot], aph);
                ptx::tc_fence_after();
                if (leader && j == 0 && li < 5) g8_stamp(p, li * 6 + 2);
                if (leader) g8_cstamp(p, cg, 3);
                if (leader) {
                    const uint32_t a_hi = tmem_base + BN + slot * Cfg::CHUNK_COLS;
                    const uint32_t a_lo = a_hi + Cfg::HALF_COLS;
                    const uint64_t sb = db0 + (uint64_t)(s * STG16) + (j % Cfg::CPS) * (G8_CK * Cfg::EB / 16);
#pragma unroll
                    for (int u = 0; u < G8_CK / Cfg::UK && !(p.debug & 4); ++u) {
                        const uint64_t dbh = sb + 2 * u, dbl = dbh + BLO16;
                        const uint32_t first = (kr > 0 || u > 0) ? 1u : 0u;
                        ptx::umma_ts<BF16>(tmem_base, a_lo + u * 8, dbh, idesc, first);
                        ptx::umma_ts<BF16>(tmem_base, a_hi + u * 8, dbl, idesc, 1u);
                        ptx::umma_ts<BF16>(tmem_base, a_hi + u * 8, dbh, idesc, 1u);
                    }
                    ptx::umma_commit(&a_empty[slot]);
                    if (j % Cfg::CPS == Cfg::CPS - 1 || kc == k_hi - 1) ptx::umma_commit(&b_empty[s]);
                }
                __syncwarp();
                if (++slot == p.ring) {
                    slot = 0;
                    aph ^= 1;
                }
                if ((j % Cfg::CPS == Cfg::CPS - 1 || kc == k_hi - 1) && ++s == p.bstages) {
                    s = 0;
                    bph ^= 1;
                }
                if (++kr == p.range_chunks) kr = 0;
            }
            if (leader) ptx::umma_commit(acc_full);
            if (leader && li < 5) g8_stamp(p, li * 6 + 3);
            __syncwarp();
            ++i;
        }
    }

    ptx::tc_fence_before();
    __syncthreads();
    if (threadIdx.x == 0) g8_stamp(p, 30);
    if (warp == G8_MMA_WARP) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem_base, G8_TMEM_COLS);
    }
}

// ----------------------------------------------------------------------------------------
// Host side
// ----------------------------------------------------------------------------------------
static PFN_cuTensorMapEncodeTiled_v12000 g8_encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
                cudaSuccess && q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
    });
    return fn;
}

template <int BN, bool BF16>
static int launch_g8_cfg(const G8Params& prm_in, const void* w_hi, const void* w_lo, cudaStream_t st) {
    using Cfg = G8Cfg<BN, BF16>;
    G8Params prm = prm_in;
    prm.ring = (G8_TMEM_COLS - BN) / Cfg::CHUNK_COLS;
    prm.astages = 4;
    if (const char* e = env("CB_K8_ASTAGES"))  // even: each stage stays with one producer group
        prm.astages = std::max(2, std::min(G8_ASTAGES_MAX, std::atoi(e))) & ~1;
    const int ostage_bytes = 1024 + 8 * G8_OSTAGE_BYTES;  // barriers' KB + epilogue staging
    prm.bstages = std::min(8, (225 * 1024 - ostage_bytes - prm.astages * G8_ASTAGE_BYTES) / Cfg::STAGE_BYTES);
    if (const char* e = env("CB_K8_DEBUG")) prm.debug = std::atoi(e);
    if (const char* e = env("CB_K8_BSTAGES")) prm.bstages = std::max(2, std::min(prm.bstages, std::atoi(e)));
    if (prm.bstages < 2) return fail(CB_ERR_UNSUPPORTED, "K8: shared memory for 2 weight stages");
    if (8 * (2 * prm.bstages + 2 * prm.ring + 4 + 2 * prm.astages) > 1024)
        return fail(CB_ERR_UNSUPPORTED, "K8: barrier block overflow");
    const size_t smem = 1024 + (size_t)prm.bstages * Cfg::STAGE_BYTES + prm.astages * G8_ASTAGE_BYTES +
                        ostage_bytes;
    auto kern = gemm_ts_kernel<BN, BF16>;
    static std::once_flag once;
    static cudaError_t attr_err = cudaSuccess;
    std::call_once(once, [&] {
        attr_err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    });
    if (attr_err != cudaSuccess)
        return fail(CB_ERR_CUDA, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(attr_err));
    auto enc = g8_encode_fn();
    if (!enc) return fail(CB_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    if ((reinterpret_cast<uintptr_t>(w_hi) | reinterpret_cast<uintptr_t>(w_lo)) & 15)
        return fail(CB_ERR_MISALIGNED, "split weights must be 16-byte aligned");
    CUtensorMap mh, ml;
    for (int h = 0; h < 2; ++h) {
        cuuint64_t dims[2] = {(cuuint64_t)prm.g.kdim_pad, (cuuint64_t)prm.g.K};
        cuuint64_t strides[1] = {(cuuint64_t)prm.g.kdim_pad * Cfg::EB};
        cuuint32_t box[2] = {(cuuint32_t)Cfg::KE, (cuuint32_t)BN};
        cuuint32_t es[2] = {1, 1};
        CUresult r = enc(h ? &ml : &mh, BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                         2, const_cast<void*>(h ? w_lo : w_hi), dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS)
            return fail(CB_ERR_CUDA, "cuTensorMapEncodeTiled (weights) failed: " + std::to_string((int)r));
    }
    CUtensorMap ma{};
    if (prm.tma_a) {  // the fp32 matrix [rows][ld], boxes of 128 pixels x 32 rows
        cuuint64_t dims[2] = {(cuuint64_t)prm.pm.src_ld, (cuuint64_t)prm.g.G * prm.g.kdim};
        cuuint64_t strides[1] = {(cuuint64_t)prm.pm.src_ld * 4};
        cuuint32_t box[2] = {(cuuint32_t)G8_BM, (cuuint32_t)G8_CK};
        cuuint32_t es[2] = {1, 1};
        CUresult r = enc(&ma, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(prm.src), dims,
                         strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS)
            return fail(CB_ERR_CUDA, "cuTensorMapEncodeTiled (A) failed: " + std::to_string((int)r));
    }
    if (prm.tail_k) {
        // the K parts wait on each other: every CTA of the grid must be resident at once
        int per_sm = 0;
        const size_t smem_launch = std::max<size_t>(smem, 120 * 1024);
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, G8_THREADS, smem_launch) != cudaSuccess ||
            (int64_t)per_sm * sm_count() < std::min<int64_t>(prm.items, sm_count())) {
            (void)cudaGetLastError();
            prm.items = prm.full_items + (prm.items - prm.full_items) / prm.tail_split;  // no split
            prm.full_items = prm.items;
            prm.tail_split = 1;
            prm.tail_k = 0;
        } else {
            const int64_t tail_tiles = (prm.items - prm.full_items) / prm.tail_split;
            const uint32_t need = (uint32_t)(tail_tiles * (BN / 32) * 4);
            static std::mutex mu;
            static uint32_t next = 0;
            static uint32_t* pool = nullptr;
            std::lock_guard<std::mutex> lk(mu);
            if (!pool && cudaGetSymbolAddress(reinterpret_cast<void**>(&pool), g8_flags) != cudaSuccess)
                return fail(CB_ERR_CUDA, "cudaGetSymbolAddress(g8_flags)");
            if (need > (uint32_t)G8_FLAG_SLOTS) return fail(CB_ERR_UNSUPPORTED, "K8: too many tail tiles");
            if (next + need > (uint32_t)G8_FLAG_SLOTS) next = 0;
            prm.flags = pool + next;
            next += need;
        }
    }
    CUtensorMap my{};
    if (prm.tma_y) {  // NCHW y {PQ, K, N} or an output matrix {ld, K, 1}, 32 x 32 boxes
        const bool nchw = prm.tma_y == 1;
        const cuuint64_t inner = nchw ? (cuuint64_t)prm.g.PQ : (cuuint64_t)prm.pm.dst_ld;
        const cuuint64_t outer = nchw ? (cuuint64_t)prm.g.N : 1;
        cuuint64_t dims[3] = {inner, (cuuint64_t)prm.g.K, outer};
        cuuint64_t strides[2] = {inner * 4, inner * prm.g.K * 4};
        cuuint32_t box[3] = {32, 32, 1};
        cuuint32_t es[3] = {1, 1, 1};
        CUresult r = enc(&my, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, prm.out, dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                         CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) prm.tma_y = 0;  // per-lane stores
    }
    const int grid = (int)std::min<int64_t>(prm.items, sm_count());
    if (env("CB_K8_TRACE")) prm.trace = debug_trace_buffer(1024, st);  // + chunk stamps
    kern<<<grid, G8_THREADS, std::max<size_t>(smem, 120 * 1024), st>>>(prm, mh, ml, ma, my);
    return check_launch("gemm_ts_kernel");
}

// Matrix / slice sources only (the stepwise GEMMs).  Returns CB_ERR_UNSUPPORTED when the
// caller should fall back to K4.
int launch_gemm_ts(bool bf16, const Geom& g, const PixMap& pm, const float* src, const void* w_hi,
                   const void* w_lo, const float* bias, float* out, int add_mode, cudaStream_t st) {
    if (pm.src_mode == SRC_CONV || env("CB_NO_K8")) return CB_ERR_UNSUPPORTED;
    if (pm.j_count == 0) return CB_OK;
    G8Params prm{};
    prm.g = g;
    prm.pm = pm;
    prm.src = src;
    prm.bias = add_mode ? nullptr : bias;
    prm.out = out;
    prm.add_mode = add_mode;
    prm.nchunks = (g.kdim + G8_CK - 1) / G8_CK;
    {  // balanced accumulator ranges of at most promote_k elements
        const int rc = std::max(1, promote_k(bf16) / G8_CK);
        const int nr = (prm.nchunks + rc - 1) / rc;
        prm.range_chunks = std::max(1, (prm.nchunks + nr - 1) / nr);
    }
    int bn = g.kpg <= 64 ? 64 : g.kpg <= 128 ? 128 : 256;
    if (const char* e = env("CB_K8_BN")) bn = std::min(bn, std::max(64, std::atoi(e)));  // diagnostics
    prm.m_tiles = (pm.j_count + G8_BM - 1) / G8_BM;
    // (narrower channel tiles for short grids measured slower: A is rebuilt per channel tile)
    prm.n_tiles = (g.kpg + bn - 1) / bn;
    prm.items = prm.m_tiles * prm.n_tiles * g.G;
    prm.full_items = prm.items;
    prm.tail_split = 1;
    {
        const int64_t grid = std::min<int64_t>(prm.items, sm_count());
        const int64_t tail = prm.items % grid;
        static const bool no_split = std::getenv("CB_K8_NO_TAIL_SPLIT") != nullptr;
        // K split on request (CB_K8_KSPLIT = max parts, read per launch).  Measured on cfg4
        // (3xBF16): the tail's MMAs drop from 31 to 14-21 us, but the parts' ordered
        // read-add-store epilogues (~1.7 TB/s of NCHW stores chip-wide) give it all back:
        // 94-98 us either way, so the channel split stays the default.
        const char* ks = env("CB_K8_KSPLIT");
        const int kmax = ks ? std::atoi(ks) : 0;
        const int kparts = (int)std::min<int64_t>(std::min<int64_t>(grid / std::max<int64_t>(tail, 1), kmax),
                                                  prm.nchunks / 4);
        if (!no_split && prm.items > grid && tail > 0 && kparts >= 2 &&
            (prm.nchunks + kparts - 1) / kparts <= prm.range_chunks) {
            prm.full_items = prm.items - tail;
            prm.tail_split = kparts;
            prm.tail_k = 1;
            prm.items = prm.full_items + tail * kparts;
        } else if (!no_split && prm.items > grid && tail > 0) {
            // parts of 32+ channels that hold real output channels (a part past kpg would
            // have nothing to store)
            const int parts = (int)std::min<int64_t>(std::min<int64_t>(grid / tail, 4),
                                                     (std::min(bn, g.kpg) + 31) / 32);
            if (parts >= 2) {
                prm.full_items = prm.items - tail;
                prm.tail_split = parts;
                prm.items = prm.full_items + tail * parts;
            }
        }
    }
    prm.tma_a = pm.src_mode == SRC_MATRIX && (pm.src_ld % 4) == 0 &&
                (reinterpret_cast<uintptr_t>(src) & 15) == 0 && pm.j_begin + pm.j_count <= pm.src_ld &&
                !env("CB_K8_NO_TMA_A");
    // TMA-store epilogue: NCHW y (the Im2col-GEMM drop-in) or an output matrix (the SConv
    // accumulators, cb_gemm); 16-byte row strides and base
    prm.tma_y = 0;
    if (!env("CB_K8_NO_TMA_STORE") && (reinterpret_cast<uintptr_t>(out) & 15) == 0 && !add_mode) {
        if (pm.dst_mode == DST_NCHW && g.PQ % 4 == 0 && pm.j_begin == 0)
            prm.tma_y = 1;
        else if (pm.dst_mode == DST_MATRIX && pm.dst_ld % 4 == 0)
            prm.tma_y = 2;
    }
    switch (bn) {
        case 64: return bf16 ? launch_g8_cfg<64, true>(prm, w_hi, w_lo, st) : launch_g8_cfg<64, false>(prm, w_hi, w_lo, st);
        case 128: return bf16 ? launch_g8_cfg<128, true>(prm, w_hi, w_lo, st) : launch_g8_cfg<128, false>(prm, w_hi, w_lo, st);
        default: return bf16 ? launch_g8_cfg<256, true>(prm, w_hi, w_lo, st) : launch_g8_cfg<256, false>(prm, w_hi, w_lo, st);
    }
}

}  // namespace cb
