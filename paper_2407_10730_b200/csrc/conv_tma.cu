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
// CG = 1: one CTA per 128-pixel tile.  CG = 2: a CTA pair (cluster of 2, cta_group::2)
// owns a 256-pixel tile: each CTA loads its own 128 pixel rows and half of the BN weight
// rows, the leader issues M=256 MMAs that read both CTAs' shared memory, and each CTA's
// TMEM holds the accumulator rows of its pixels.  Per MMA cycle this halves the operand
// bytes each SM pulls from L2, which is what bounds the CG = 1 kernel (ncu, profiles/).
//
// CTA layout (192 threads, persistent over a static tile schedule, 1 CTA / SM):
//   warps 0..3  epilogue: tcgen05.ld 32 columns at a time -> +bias -> coalesced NCHW stores
//               (lane = pixel, so each store instruction of a warp writes 32 consecutive
//               pixels of one output channel) or fp32 reductions for split-K.
//   warp 4      TMA producer (one elected lane; both CTAs of a pair)
//   warp 5      TMEM allocator (2 x BN columns: double-buffered accumulator) + MMA issuer
//               (leader CTA only)
// Barriers: full/empty per smem stage (TMA tx-count on the leader / tcgen05.commit
// multicast to both CTAs), tmem_full / tmem_empty per accumulator buffer (the leader's
// tmem_empty collects all 128*CG epilogue threads), so the epilogue of tile i overlaps the
// MMAs of tile i+1.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <mutex>

#include "cb_common.cuh"
#include "sm100_ptx.cuh"

namespace cb {

constexpr int TMA_THREADS = 192;
constexpr int TMA_BM = 128;  // pixel rows per CTA
// Warp roles.  The issue arbiter favours higher warp ids and warp w runs on SMSP w % 4, so
// the latency-critical TMA and MMA warps take the highest ids and win their SMSP against
// the epilogue warps sharing it (epilogue warp q must be warp q mod 4 to reach TMEM lane
// quadrant q).
constexpr int PRODUCER_WARP = 4;
constexpr int MMA_WARP = 5;

struct TmaParams {
    Geom g;
    FusedLayout L;
    const float* bias;
    float* out;
    int n_tiles;          // output-channel tiles per group
    int64_t m_tiles;      // pixel tiles of 128*CG
    int splits;
    int kb_per_split;
    int64_t total_tiles;  // n_tiles * m_tiles * G * splits
    int add_mode;         // 0: store acc + bias, 1: fp32 reduction into out
    int tma_store;        // 1: epilogue stages 32-channel chunks in smem, TMA-stores y (tm_y)
    int bulk_parts;       // 1: tail parts write their partial chunks with 1-D bulk copies
    int out_al16;         // 1: y is 16-byte aligned (the tail fixup's float4 stores need it)
    // Accumulator promotion (see promote_k): an item's K blocks run as ranges of at most
    // range_kb blocks, each into a fresh TMEM accumulator (the double buffer alternates); the
    // epilogue adds range partials in fp32 -- into y for whole tiles, into the part's slab
    // for tail parts -- so no accumulator sums more than ~promote_k reduction elements.
    int range_kb;
    // Tail split-K ("stream-K lite"): the first full_items work items are whole tiles;
    // the tail_tiles tiles of the last, partial wave are each cut into tail_parts K
    // ranges of tail_kbp stages so every cluster gets work.  Parts write fp32 partials to
    // `partials`; the last part to arrive (per-tile counter) sums them in part order,
    // adds the bias and stores the tile, so the result is deterministic.
    int64_t full_items;
    int tail_tiles, tail_parts, tail_kbp;
    int64_t total_items;
    int tail_last;        // diagnostics (CB_TMA_TAIL_LAST): the old order, tail parts last
    int* counters;        // 2 * tail_tiles * CG ([written][done]), self-resetting
    float* partials;      // tail_tiles * tail_parts * CG * BN * 128
    unsigned long long* trace;  // diagnostics (CB_TMA_TRACE): per-CTA globaltimer stamps
    int debug;            // diagnostics only (CB_TMA_DEBUG): 1 = skip operand loads,
                          // 2 = skip epilogue stores, 3 = both.  Results are garbage.
};

constexpr int TRACE_SLOTS = 32;
constexpr int MAX_TAIL_OTHERS = 3;  // over-full grids: tail tiles split into at most 4 K parts
constexpr int MAX_SHORT_PARTS = 16;  // short grids (tiles < clusters) with long reductions
__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void trace_stamp(const TmaParams& p, int slot) {
    if (kTrace && p.trace && slot < TRACE_SLOTS) p.trace[blockIdx.x * TRACE_SLOTS + slot] = globaltimer();
}

template <int BN, int STAGES, bool BF16, int CG>
struct TmaCfg {
    static constexpr int EB = BF16 ? 2 : 4;
    static constexpr int KE = 128 / EB;              // reduction elements per stage
    static constexpr int B_ROWS = BN / CG;           // weight rows this CTA loads
    static constexpr int A_BYTES = TMA_BM * 128;     // one of A_hi / A_lo
    static constexpr int B_BYTES = B_ROWS * 128;     // one of B_hi / B_lo
    static constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;
    static constexpr int OSTAGE_BYTES = 2 * 32 * TMA_BM * 4;  // epilogue: 2 x [32 ch][128 px] fp32
    static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + OSTAGE_BYTES + 1024 + 256;
    static constexpr uint32_t TMEM_COLS = 2 * BN;
    static_assert(SMEM_BYTES <= 232448, "shared memory budget");
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

struct WorkItem {
    int nt, gi, kb0, kb1;
    int64_t mt;
    int tail;   // tail-tile index, or -1 for a whole tile
    int part;   // K part of a tail tile
};

// Item order: the tail parts come FIRST (items [0, tail_items), at most one per cluster, all
// concurrent), whole tiles after them.  A part's fixup -- park, wait for the other parts,
// sum its own chunks -- then runs in the epilogue warps while the MMA warp is already on the
// cluster's next whole tile (the other TMEM accumulator), instead of trailing the kernel.
__device__ __forceinline__ WorkItem decode_item(const TmaParams& p, int64_t i) {
    WorkItem w;
    int ks;
    const int64_t tail_items = p.total_items - p.full_items;
    if (!p.tail_last) i = i < tail_items ? p.full_items + i : i - tail_items;
    if (i < p.full_items) {
        decode_tile(p, i, w.nt, w.mt, w.gi, ks);
        w.kb0 = ks * p.kb_per_split;
        w.kb1 = min(p.L.num_kb, w.kb0 + p.kb_per_split);
        w.tail = -1;
        w.part = 0;
    } else {
        const int64_t j = i - p.full_items;
        w.tail = (int)(j / p.tail_parts);
        w.part = (int)(j - (int64_t)w.tail * p.tail_parts);
        decode_tile(p, p.full_items + w.tail, w.nt, w.mt, w.gi, ks);
        w.kb0 = w.part * p.tail_kbp;
        w.kb1 = min(p.L.num_kb, w.kb0 + p.tail_kbp);
    }
    return w;
}

// accumulator ranges of an item's K blocks [kb0, kb1): nr balanced ranges of <= range_kb
__device__ __forceinline__ int n_ranges(int kb0, int kb1, int range_kb) {
    return max(1, (kb1 - kb0 + range_kb - 1) / range_kb);
}
__device__ __forceinline__ int range_begin(int kb0, int kb1, int nr, int r) {
    return kb0 + (int)((int64_t)(kb1 - kb0) * r / nr);
}

__device__ __forceinline__ void epi_barrier() {  // the 128 epilogue threads (warps 0..3)
    asm volatile("bar.sync 1, 128;" ::: "memory");
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

template <int BN, int STAGES, bool BF16, int CG>
__global__ void __launch_bounds__(TMA_THREADS, 1)
conv_tma_kernel(const __grid_constant__ TmaParams p, const __grid_constant__ CUtensorMap tm_ahi,
                const __grid_constant__ CUtensorMap tm_alo,
                const __grid_constant__ CUtensorMap tm_bhi,
                const __grid_constant__ CUtensorMap tm_blo,
                const __grid_constant__ CUtensorMap tm_y) {
    using Cfg = TmaCfg<BN, STAGES, BF16, CG>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    float* ostage = reinterpret_cast<float*>(smem + STAGES * Cfg::STAGE_BYTES);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * Cfg::STAGE_BYTES + Cfg::OSTAGE_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const Geom& g = p.g;
    const FusedLayout& L = p.L;
    const uint32_t rank = CG == 2 ? ptx::cluster_ctarank() : 0;
    const int64_t cl0 = blockIdx.x / CG;        // this CTA's cluster (tile-schedule unit)
    const int64_t ncl = gridDim.x / CG;

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            ptx::mbar_init(&tfull[a], 1);
            ptx::mbar_init(&tempty[a], 128 * CG);
        }
        ptx::fence_mbar_init();
    }
    if (warp == PRODUCER_WARP && lane == 0) {
        ptx::tma_prefetch_desc(&tm_ahi);
        ptx::tma_prefetch_desc(&tm_alo);
        ptx::tma_prefetch_desc(&tm_bhi);
        ptx::tma_prefetch_desc(&tm_blo);
    }
    if (warp == MMA_WARP) {
        if (CG == 2)
            ptx::tmem_alloc_pair(tmem_slot, Cfg::TMEM_COLS);
        else
            ptx::tmem_alloc(tmem_slot, Cfg::TMEM_COLS);
    }
    ptx::tc_fence_before();
    if (CG == 2)
        ptx::cluster_sync();
    else
        __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    // everything above overlapped the preceding kernel; its outputs (the split activations,
    // the zeroed tail counters) are read only after this point
    asm volatile("griddepcontrol.wait;" ::: "memory");

    if (warp == PRODUCER_WARP) {
        // ================================ TMA producer ==================================
        // The whole warp walks the schedule (warp-uniform values in uniform registers);
        // one elected lane issues.  The (tap, chunk) walk advances by counters.
        const uint32_t leader = ptx::elect_one();
        int stage = 0;
        uint32_t phase = 0;
        constexpr uint32_t tx = CG * (2 * Cfg::A_BYTES + 2 * Cfg::B_BYTES);
        for (int64_t t = cl0; t < p.total_items; t += ncl) {
            const WorkItem it = decode_item(p, t);
            const int gi = it.gi;
            const int64_t m0 = it.mt * (TMA_BM * CG) + rank * TMA_BM;
            const int n0 = (int)(m0 / g.PQ);
            const int rem = (int)(m0 - (int64_t)n0 * g.PQ);
            const int oy0 = rem / g.Q, ox0 = rem - (rem / g.Q) * g.Q;
            const int wc = ox0 * g.sw - g.pw, hc = oy0 * g.sh - g.ph;
            const int brow = gi * g.kpg + it.nt * BN + (int)rank * Cfg::B_ROWS;
            int q = it.kb0 * L.cps;  // chunk index = (r*S + s)*chk + cbi
            int tap = q / L.chk;
            int cbi = q - tap * L.chk;
            int r = tap / g.S;
            int s = tap - r * g.S;
            for (int kb = it.kb0; kb < it.kb1; ++kb) {
                ptx::mbar_wait(&empty[stage], phase ^ 1);
                uint8_t* st = smem + stage * Cfg::STAGE_BYTES;
                if (p.debug & 1) {  // diagnostics: MMA-only timing, no operand traffic
                    if (leader && rank == 0) ptx::mbar_arrive(&full[stage]);
                    __syncwarp();
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                    continue;
                }
                if (leader && rank == 0) ptx::mbar_arrive_expect_tx(&full[stage], tx);
                const uint32_t lbar = ptx::leader_bar(&full[stage]);
                for (int i = 0; i < L.cps; ++i, ++q) {
                    int c = L.c_alloc, offw = 0, offh = 0;  // past the end: all-OOB zeros
                    if (q < L.total_chunks) {
                        c = gi * g.cpg + cbi * L.cb;
                        offw = s * g.dw;
                        offh = r * g.dh;
                    }
                    const int off = i * TMA_BM * L.chunk_bytes;
                    if (leader) {
                        if (CG == 2) {
                            ptx::tma_load_im2col_4d_pair(st + off, &tm_ahi, lbar, c, wc, hc, n0,
                                                         (uint16_t)offw, (uint16_t)offh);
                            ptx::tma_load_im2col_4d_pair(st + Cfg::A_BYTES + off, &tm_alo, lbar, c,
                                                         wc, hc, n0, (uint16_t)offw, (uint16_t)offh);
                        } else {
                            ptx::tma_load_im2col_4d(st + off, &tm_ahi, &full[stage], c, wc, hc, n0,
                                                    (uint16_t)offw, (uint16_t)offh);
                            ptx::tma_load_im2col_4d(st + Cfg::A_BYTES + off, &tm_alo, &full[stage],
                                                    c, wc, hc, n0, (uint16_t)offw, (uint16_t)offh);
                        }
                    }
                    if (++cbi == L.chk) {
                        cbi = 0;
                        if (++s == g.S) {
                            s = 0;
                            ++r;
                        }
                    }
                }
                uint8_t* bdst = st + 2 * Cfg::A_BYTES;
                if (leader) {
                    if (CG == 2) {
                        ptx::tma_load_2d_pair(bdst, &tm_bhi, lbar, kb * Cfg::KE, brow);
                        ptx::tma_load_2d_pair(bdst + Cfg::B_BYTES, &tm_blo, lbar, kb * Cfg::KE, brow);
                    } else {
                        ptx::tma_load_2d(bdst, &tm_bhi, &full[stage], kb * Cfg::KE, brow);
                        ptx::tma_load_2d(bdst + Cfg::B_BYTES, &tm_blo, &full[stage], kb * Cfg::KE,
                                         brow);
                    }
                }
                __syncwarp();
                if (++stage == STAGES) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
    } else if (warp == MMA_WARP) {
        // ============================ MMA issuer (leader CTA) =============================
        // Whole warp walks the schedule; descriptors are the stage-0 descriptors plus
        // constant offsets (the 14-bit address field never carries inside smem); one
        // elected lane issues the 12 MMAs of a K block and the commits.
        if (rank == 0) {
            constexpr uint32_t idesc = ptx::idesc_f32acc<BF16>(TMA_BM * CG, BN);
            constexpr uint32_t STG16 = Cfg::STAGE_BYTES >> 4;
            constexpr uint32_t ALO16 = Cfg::A_BYTES >> 4, BLO16 = Cfg::B_BYTES >> 4;
            const uint32_t s0 = ptx::smem_u32(smem);
            const uint64_t da0 = a_desc(s0, L.chunk_bytes, 0);
            uint32_t aoff[4];
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) aoff[kk] = (uint32_t)(a_desc(s0, L.chunk_bytes, kk) - da0);
            const uint64_t db0 = ptx::sdesc_k_sw128(s0 + 2 * Cfg::A_BYTES);
            const uint32_t leader = ptx::elect_one();
            int stage = 0;
            uint32_t phase = 0;
            int local = 0;
            for (int64_t t = cl0; t < p.total_items; t += ncl) {
                const WorkItem it = decode_item(p, t);
                const int nr = n_ranges(it.kb0, it.kb1, p.range_kb);
#pragma unroll 1
                for (int rg = 0; rg < nr; ++rg, ++local) {
                const int rkb0 = range_begin(it.kb0, it.kb1, nr, rg);
                const int rkb1 = range_begin(it.kb0, it.kb1, nr, rg + 1);
                const int acc = local & 1;
                const uint32_t acc_phase = (local >> 1) & 1;
                ptx::mbar_wait(&tempty[acc], acc_phase ^ 1);
                ptx::tc_fence_after();
                const uint32_t d = tmem_base + acc * BN;
                for (int kb = rkb0; kb < rkb1; ++kb) {
                    ptx::mbar_wait(&full[stage], phase);
                    ptx::tc_fence_after();
                    const uint64_t sa = da0 + (uint64_t)(stage * STG16);
                    const uint64_t sb = db0 + (uint64_t)(stage * STG16);
                    if (leader) {
#pragma unroll
                        for (int kk = 0; kk < 4; ++kk) {
                            const uint64_t dah = sa + aoff[kk];
                            const uint64_t dal = dah + ALO16;
                            const uint64_t dbh = sb + 2 * kk;
                            const uint64_t dbl = dbh + BLO16;
                            const uint32_t first = (kb != rkb0 || kk != 0) ? 1u : 0u;
                            if (CG == 2) {
                                ptx::umma_pair<BF16>(d, dal, dbh, idesc, first);
                                ptx::umma_pair<BF16>(d, dah, dbl, idesc, 1);
                                ptx::umma_pair<BF16>(d, dah, dbh, idesc, 1);
                            } else {
                                ptx::umma<BF16>(d, dal, dbh, idesc, first);
                                ptx::umma<BF16>(d, dah, dbl, idesc, 1);
                                ptx::umma<BF16>(d, dah, dbh, idesc, 1);
                            }
                        }
                        if (CG == 2)
                            ptx::umma_commit_pair(&empty[stage]);
                        else
                            ptx::umma_commit(&empty[stage]);
                    }
                    __syncwarp();
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                if (leader) {
                    if (CG == 2)
                        ptx::umma_commit_pair(&tfull[acc]);
                    else
                        ptx::umma_commit(&tfull[acc]);
                }
                __syncwarp();
                }
            }
        }
    } else {
        // ========================== epilogue (warps 0..3) ==============================
        const int quad = warp;               // TMEM lane quadrant this warp may access
        const int row = quad * 32 + lane;    // pixel row within this CTA's 128 rows
        const uint32_t tempty_leader0 =
            CG == 2 ? ptx::mapa_shared(ptx::smem_u32(&tempty[0]), 0) : 0;
        int local = 0;
        int ochunk = 0;  // staged output chunks (double-buffered ostage)
        for (int64_t t = cl0; t < p.total_items; t += ncl, ++local) {
            const WorkItem it = decode_item(p, t);
            const int gi = it.gi;
            const int64_t j = it.mt * (TMA_BM * CG) + rank * TMA_BM + row;
            const bool jvalid = j < g.npix;
            int64_t obase = 0;
            if (jvalid) {
                const int64_t n = j / g.PQ;
                obase = n * (int64_t)g.K * g.PQ + (j - n * g.PQ);
            }
            const int f_tile0 = it.nt * BN;
            const bool do_store = jvalid && !(p.debug & 2);
            float* dst = p.out + obase + (int64_t)(gi * g.kpg + f_tile0) * g.PQ;
            const float* bias = p.bias ? p.bias + gi * g.kpg + f_tile0 : nullptr;
            const int nr = n_ranges(it.kb0, it.kb1, p.range_kb);
            const bool promoted = nr > 1;
            const int nch_all = (min(BN, g.kpg - f_tile0) + 31) / 32;
            // this CTA's fp32 slab of a tail part ([ch/4][row][ch%4], see the fixup below)
            float* const part_slab = it.tail >= 0
                ? p.partials + ((int64_t)it.tail * p.tail_parts * CG + rank) * ((int64_t)BN * TMA_BM) +
                      (int64_t)it.part * CG * ((int64_t)BN * TMA_BM)
                : nullptr;
            // ---- non-final accumulator ranges: fold each partial into fp32 storage (whole
            // tiles: y, bias with the first range; tail parts: the part's own slab) ----
#pragma unroll 1
            for (int rg = 0; rg + 1 < nr; ++rg, ++local) {
                const int acc = local & 1;
                ptx::mbar_wait(&tfull[acc], (local >> 1) & 1);
                ptx::tc_fence_after();
#pragma unroll 1
                for (int ci = 0; ci < nch_all; ++ci) {
                    const int c0 = ci * 32;
                    const int nvalid = min(32, g.kpg - (f_tile0 + c0));
                    uint32_t r[32];
                    ptx::tmem_ld_32x32b_x32(tmem_base + acc * BN + ((uint32_t)(quad * 32) << 16) + c0, r);
                    ptx::tmem_ld_wait();
                    if (ci + 1 == nch_all) {
                        ptx::tc_fence_before();
                        if (CG == 2)
                            ptx::mbar_arrive_remote(tempty_leader0 + acc * sizeof(uint64_t));
                        else
                            ptx::mbar_arrive(&tempty[acc]);
                    }
                    // read-modify-writes: every load of a chunk is issued before its first
                    // store (the compiler cannot reorder a load past a possibly aliasing store,
                    // and one load round trip per element made the epilogue 10x slower)
                    if (it.tail >= 0) {
                        float4* sl = reinterpret_cast<float4*>(part_slab) + (int64_t)(ci * 8) * TMA_BM + row;
                        float4 o[8];
#pragma unroll
                        for (int q = 0; q < 8; ++q)
                            o[q] = rg > 0 ? __ldcg(sl + (int64_t)q * TMA_BM) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                        for (int q = 0; q < 8; ++q)
                            __stcg(sl + (int64_t)q * TMA_BM,
                                   make_float4(__uint_as_float(r[4 * q]) + o[q].x, __uint_as_float(r[4 * q + 1]) + o[q].y,
                                               __uint_as_float(r[4 * q + 2]) + o[q].z, __uint_as_float(r[4 * q + 3]) + o[q].w));
                    } else if (do_store) {
                        float* d = dst + (int64_t)c0 * g.PQ;
                        if (p.add_mode) {
#pragma unroll
                            for (int i = 0; i < 32; ++i)
                                if (i < nvalid) atomicAdd(d + (int64_t)i * g.PQ, __uint_as_float(r[i]));
                        } else {
                            float o[32];
#pragma unroll
                            for (int i = 0; i < 32; ++i)
                                o[i] = i >= nvalid ? 0.f : rg > 0 ? __ldcg(d + (int64_t)i * g.PQ)
                                                     : (bias ? __ldg(bias + c0 + i) : 0.f);
#pragma unroll
                            for (int i = 0; i < 32; ++i)
                                if (i < nvalid) d[(int64_t)i * g.PQ] = __uint_as_float(r[i]) + o[i];
                        }
                    }
                }
            }
            const int acc = local & 1;
            const uint32_t acc_phase = (local >> 1) & 1;
            if (local == 0 && threadIdx.x == 0) trace_stamp(p, 0);
            ptx::mbar_wait(&tfull[acc], acc_phase);
            ptx::tc_fence_after();
            if (threadIdx.x == 0) trace_stamp(p, 1 + local);  // accumulator ready

            if (it.tail >= 0) {
                // ---- tail split-K, symmetric fixup: the P parts of a tail tile run
                // concurrently on distinct co-resident clusters; part p owns the 32-channel
                // chunks [P*p/.., ..) of the tile.  Every part parks the chunks it does not
                // own as fp32 partials ([channel][row]: each warp access one 128-byte line),
                // publishes, waits for all P, then sums its own chunks over the parts in part
                // order (deterministic) and stores them.  Counters: [written][done] per
                // (tail tile, CTA rank); the last part through `done` resets both. ----
                const int P = p.tail_parts;
                const int64_t slab = (int64_t)BN * TMA_BM;
                const int nch = (min(BN, g.kpg - f_tile0) + 31) / 32;
                const int own_lo = it.part * nch / P, own_hi = (it.part + 1) * nch / P;
                // partial slab layout [ch / 4][row][ch % 4]: a thread's 4 consecutive channels
                // are one float4 and a warp's float4 accesses are one 512-byte run
                float* slab_of = p.partials + ((int64_t)it.tail * P * CG + rank) * slab;  // + q*CG*slab
                int* written = p.counters + 2 * (it.tail * CG + rank);
                int* done = written + 1;
                const uint32_t lane_tm = tmem_base + acc * BN + ((uint32_t)(quad * 32) << 16);
                float* mine = slab_of + (int64_t)it.part * CG * slab;
#pragma unroll 1
                for (int ci = 0; ci < nch; ++ci) {
                    if (ci >= own_lo && ci < own_hi) continue;
                    uint32_t r[32];
                    ptx::tmem_ld_32x32b_x32(lane_tm + ci * 32, r);
                    ptx::tmem_ld_wait();
                    float4* sl = reinterpret_cast<float4*>(mine) + (int64_t)(ci * 8) * TMA_BM + row;
                    float4 o[8];  // the part's earlier ranges, folded into its slab (loads first)
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        o[j] = promoted ? __ldcg(sl + (int64_t)j * TMA_BM) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        __stcg(sl + (int64_t)j * TMA_BM,
                               make_float4(__uint_as_float(r[4 * j]) + o[j].x, __uint_as_float(r[4 * j + 1]) + o[j].y,
                                           __uint_as_float(r[4 * j + 2]) + o[j].z, __uint_as_float(r[4 * j + 3]) + o[j].w));
                }
                if (threadIdx.x == 0) trace_stamp(p, 20);  // partials written (issued)
                __threadfence();
                epi_barrier();
                if (threadIdx.x == 0) {
                    atomicAdd(written, 1);
                    trace_stamp(p, 22);  // waiting for the other parts
                    while (*reinterpret_cast<volatile int*>(written) < P) __nanosleep(64);
                    trace_stamp(p, 23);  // all parts published
                }
                epi_barrier();
                __threadfence();
                // own chunks: all other parts' values of a chunk are loaded before any of its
                // stores issue (loads never queue behind stores in L1)
                // Vector stores (PQ % 4 == 0: a group of 4 pixels never straddles an image):
                // lane l of the epilogue stores pixels m0 + 4l .. + 3 of channel rows.
                const bool vec_store = (g.PQ % 4) == 0 && p.out_al16 && !(p.debug & 2);
                const int64_t jv = it.mt * (TMA_BM * CG) + rank * TMA_BM + 4 * lane;
                const bool gvalid = jv < g.npix;
                float* vbase = p.out;
                if (vec_store && gvalid) {
                    const int64_t nv = jv / g.PQ;
                    vbase += nv * (int64_t)g.K * g.PQ + (jv - nv * g.PQ) + (int64_t)(gi * g.kpg + f_tile0) * g.PQ;
                }
#pragma unroll 1
                for (int ci = own_lo; ci < own_hi; ++ci) {
                    const int c0 = ci * 32;
                    const int nvalid = min(32, g.kpg - (f_tile0 + c0));
                    uint32_t r[32];
                    ptx::tmem_ld_32x32b_x32(lane_tm + c0, r);
                    // every other part's values of the chunk in flight at once (one L2
                    // round trip per chunk), then the sum in part order
                    // parts in groups of 4: every other part's values of a group in flight at
                    // once (one L2 round trip per group), summed in part order
                    ptx::tmem_ld_wait();
                    float v[32];
#pragma unroll
                    for (int i = 0; i < 32; ++i) v[i] = 0.f;
#pragma unroll 1
                    for (int q0 = 0; q0 < P; q0 += 4) {
                        float4 pv[4][8];
#pragma unroll
                        for (int o = 0; o < 4; ++o) {
                            const int q = q0 + o;
                            if (q < P && (q != it.part || promoted)) {
                                const float4* src = reinterpret_cast<const float4*>(
                                                        slab_of + (int64_t)q * CG * slab) +
                                                    (int64_t)(ci * 8) * TMA_BM + row;
#pragma unroll
                                for (int j = 0; j < 8; ++j) pv[o][j] = __ldcg(src + (int64_t)j * TMA_BM);
                            }
                        }
#pragma unroll
                        for (int o = 0; o < 4; ++o) {
                            const int q = q0 + o;
                            if (q >= P) break;
                            if (q == it.part) {
                                float own[32];  // last range (TMEM) + earlier ranges (own slab)
#pragma unroll
                                for (int i = 0; i < 32; ++i) own[i] = __uint_as_float(r[i]);
                                if (promoted) {
#pragma unroll
                                    for (int j = 0; j < 8; ++j) {
                                        own[4 * j] += pv[o][j].x;
                                        own[4 * j + 1] += pv[o][j].y;
                                        own[4 * j + 2] += pv[o][j].z;
                                        own[4 * j + 3] += pv[o][j].w;
                                    }
                                }
#pragma unroll
                                for (int i = 0; i < 32; ++i) v[i] += own[i];
                            } else {
#pragma unroll
                                for (int j = 0; j < 8; ++j) {
                                    v[4 * j] += pv[o][j].x;
                                    v[4 * j + 1] += pv[o][j].y;
                                    v[4 * j + 2] += pv[o][j].z;
                                    v[4 * j + 3] += pv[o][j].w;
                                }
                            }
                        }
                    }
                    if (vec_store) {
                        // transpose through shared memory so each lane stores 4 consecutive
                        // pixels of one channel: a warp writes a 512-byte channel row per
                        // STG.128 instead of a 128-byte one per STG.32
                        float* buf = ostage + (ochunk & 1) * (32 * TMA_BM);
                        ++ochunk;
                        if (threadIdx.x == 0) ptx::bulk_wait_read<0>();  // no TMA store reads buf
                        epi_barrier();
#pragma unroll
                        for (int i = 0; i < 32; ++i)
                            buf[i * TMA_BM + row] = v[i] + (bias && i < nvalid ? __ldg(bias + c0 + i) : 0.f);
                        epi_barrier();
                        if (gvalid) {
#pragma unroll
                            for (int q = 0; q < 8; ++q) {
                                const int ch = quad + 4 * q;
                                if (ch < nvalid)
                                    *reinterpret_cast<float4*>(vbase + (int64_t)(c0 + ch) * g.PQ) =
                                        *reinterpret_cast<const float4*>(buf + ch * TMA_BM + 4 * lane);
                            }
                        }
                    } else if (do_store) {
                        float* d = dst + (int64_t)c0 * g.PQ;
#pragma unroll
                        for (int i = 0; i < 32; ++i)
                            if (i < nvalid)
                                d[(int64_t)i * g.PQ] = v[i] + (bias ? __ldg(bias + c0 + i) : 0.f);
                    }
                }
                ptx::tc_fence_before();
                if (CG == 2)
                    ptx::mbar_arrive_remote(tempty_leader0 + acc * sizeof(uint64_t));
                else
                    ptx::mbar_arrive(&tempty[acc]);
                if (threadIdx.x == 0) {
                    trace_stamp(p, 24);  // own chunks stored
                    if (atomicAdd(done, 1) == P - 1) {  // every part is past its wait
                        *written = 0;
                        *done = 0;
                    }
                }
                continue;
            }

            const int nchunk = (min(BN, g.kpg - f_tile0) + 31) / 32;
            // TMA store only for tiles inside one image (a box may not start at a negative
            // pixel coordinate); tiles across an image boundary store directly
            const int64_t m0t = it.mt * (TMA_BM * CG) + rank * TMA_BM;
            const int64_t n0t = m0t / g.PQ;
            const bool tile_tstore = p.tma_store && !promoted && m0t < g.npix &&
                                     (min(m0t + TMA_BM, g.npix) - 1) / g.PQ == n0t;
#pragma unroll 1
            for (int ci = 0; ci < nchunk; ++ci) {
                const int c0 = ci * 32;
                const int nvalid = min(32, g.kpg - (f_tile0 + c0));  // warp-uniform
                uint32_t r[32];
                ptx::tmem_ld_32x32b_x32(tmem_base + acc * BN + ((uint32_t)(quad * 32) << 16) + c0,
                                        r);
                ptx::tmem_ld_wait();
                if (ci + 1 == nchunk) {  // the whole accumulator is in registers: release it
                    ptx::tc_fence_before();
                    if (CG == 2)
                        ptx::mbar_arrive_remote(tempty_leader0 + acc * sizeof(uint64_t));
                    else
                        ptx::mbar_arrive(&tempty[acc]);
                }
                if (tile_tstore && !(p.debug & 2)) {
                    // stage [32 ch][128 px] (+bias) and TMA-store it (the tensor map clips
                    // the image's last tile)
                    float* buf = ostage + (ochunk & 1) * (32 * TMA_BM);
                    if (threadIdx.x == 0) ptx::bulk_wait_read<1>();
                    epi_barrier();
#pragma unroll
                    for (int i = 0; i < 32; ++i)
                        buf[i * TMA_BM + row] = __uint_as_float(r[i]) +
                                                (bias && i < nvalid ? __ldg(bias + c0 + i) : 0.f);
                    ptx::fence_proxy_async_smem();
                    epi_barrier();
                    if (threadIdx.x == 0) {
                        ptx::tma_store_3d(&tm_y, buf, (int32_t)(m0t - n0t * g.PQ),
                                          gi * g.kpg + f_tile0 + c0, (int32_t)n0t);
                        ptx::bulk_commit();
                    }
                    ++ochunk;
                } else if (do_store) {
                    if (p.add_mode) {
#pragma unroll
                        for (int i = 0; i < 32; ++i)
                            if (i < nvalid) atomicAdd(dst + (int64_t)i * g.PQ, __uint_as_float(r[i]));
                    } else if (promoted) {  // bias and the earlier ranges are in y already
                        float o[32];  // all loads before the first store
#pragma unroll
                        for (int i = 0; i < 32; ++i) o[i] = i < nvalid ? __ldcg(dst + (int64_t)i * g.PQ) : 0.f;
#pragma unroll
                        for (int i = 0; i < 32; ++i)
                            if (i < nvalid) dst[(int64_t)i * g.PQ] = __uint_as_float(r[i]) + o[i];
                    } else if (nvalid == 32 && !bias) {
#pragma unroll
                        for (int i = 0; i < 32; ++i) dst[(int64_t)i * g.PQ] = __uint_as_float(r[i]);
                    } else {
#pragma unroll
                        for (int i = 0; i < 32; ++i)
                            if (i < nvalid)
                                dst[(int64_t)i * g.PQ] =
                                    __uint_as_float(r[i]) + (bias ? __ldg(bias + c0 + i) : 0.f);
                    }
                }
                dst += (int64_t)32 * g.PQ;
            }
        }
        if (threadIdx.x == 0) {
            ptx::bulk_wait_all();  // smem sources must outlive the bulk stores
            trace_stamp(p, TRACE_SLOTS - 1);  // epilogue finished
        }
    }

    ptx::tc_fence_before();
    if (CG == 2)
        ptx::cluster_sync();
    else
        __syncthreads();
    if (warp == MMA_WARP) {
        ptx::tc_fence_after();
        if (CG == 2)
            ptx::tmem_dealloc_pair(tmem_base, Cfg::TMEM_COLS);
        else
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

static FusedLayout base_layout(const Geom& g, bool bf16) {
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

// Fold the horizontal taps into the channels when that shortens the padded reduction
// (few channels: C=3 pads each tap to a 16-byte chunk, 147 -> 392 for a 7x7 stem; folded
// it is 7 taps of 21 -> 24 channels, 147 -> 256) -- fewer MMAs and fewer, larger TMA boxes.
// Weights are repacked to match (weight_split_taps, fold) and K0 writes the folded rows.
bool ts_eligible(const Geom& g, bool bf16);

static int stack_kmax() {  // largest K for row stacking (CB_STACK_KMAX overrides; diagnostics)
    const char* e = env("CB_STACK_KMAX");
    return e ? std::atoi(e) : 32;
}

FusedLayout fused_layout(const Geom& g, bool bf16) {
    FusedLayout L = base_layout(g, bf16);
    // Few output channels, many input channels: stack the taps (see stack_geom).  The TMA
    // im2col walk would re-read every input pixel once per tap for a handful of MMA columns.
    if (g.G == 1 && g.RS > 1 && !env("CB_NO_STACK")) {
        int mode = 0;
        if (g.RS * g.K <= 256 && g.C >= 128) mode = 1;                          // all taps
        else if (g.S > 1 && g.S * g.K <= 256 && g.K <= stack_kmax() && g.C >= 64) mode = 2;  // row taps
        if (mode) {
            FusedLayout T = base_layout(stack_geom(g, mode), bf16);
            if (T.tma) {
                T.stack = mode;
                return T;
            }
        }
    }
    // Few channels (C <= 16): the direct kernel builds A in TMEM from TMA-staged fp32 rows
    // (no activation pre-pass, no padded taps).  The tf32 split only for the compile-time
    // reduction layouts (one A buffer in TMEM instead of two).
    if (g.C <= 16 && !env("CB_NO_TS") && !(env("CB_NO_TS_TF32") && !bf16) && ts_eligible(g, bf16)) {
        FusedLayout T = L;
        T.tma = 0;
        T.fold = 0;
        T.ts = 1;
        return T;
    }
    if (env("CB_FORCE_GATHER")) {  // diagnostics: the K4 gather path (no workspace)
        L.tma = 0;
        return L;
    }
    if (g.G == 1 && g.S > 1 && g.C * g.S <= 128 && !env("CB_NO_FOLD")) {
        FusedLayout F = base_layout(fold_geom(g), bf16);
        if (F.tma && (!L.tma || F.num_kb < L.num_kb)) {
            F.fold = g.S;
            return F;
        }
    }
    return L;
}

struct TmaPlan {
    int cg, bn, stages, splits, kb_per_split, n_tiles;
    int64_t m_tiles, total_tiles;
    int grid;  // CTAs (a multiple of cg)
    // tail split-K (see TmaParams)
    int64_t full_items, total_items;
    int tail_tiles, tail_parts, tail_kbp;
};

// Cost model per candidate (cg, bn): waves over the persistent units times the per-tile
// time, which is the slower of the MMA issue time and the operand bytes the CTA pulls at
// the L2->SM rate the CG=1 kernel sustained under ncu (~40 B/cycle/SM).
// K parts of each tail tile (1 = no split): parts <= units / tail so every part has its own
// cluster (an owner spins on its parts); >= min K blocks per part; at most 4 on an over-full
// grid, 16 on a short one; and only when the MMA time a split takes off a tile exceeds the
// fixup's cost (park, publish, wait, sum: 2-3 us; cfg1 / cfg2b are faster unsplit).
static int tail_split_parts(int64_t tiles, int units, int num_kb, int bn) {
    const int64_t tail = tiles % units;
    if (tail == 0) return 1;
    const int min_kbp = tiles > units ? 4 : 2;
    int parts = (int)std::min<int64_t>(std::min<int64_t>(units / tail, num_kb / min_kbp),
                                       tiles > units ? MAX_TAIL_OTHERS + 1 : MAX_SHORT_PARTS);
    const double tile_mma = 12.0 * num_kb * (bn / 2.0);  // cycles, as in plan_tma's model
    if (parts >= 2 && tile_mma * (1.0 - 1.0 / parts) < 4000.0 && !env("CB_TMA_TAIL_ALWAYS"))
        parts = 1;
    if (parts < 2) return 1;
    const int kbp = (num_kb + parts - 1) / parts;
    return (num_kb + kbp - 1) / kbp;
}

static TmaPlan plan_tma(const Geom& g, const FusedLayout& L) {
    const int sms = sm_count();
    const char* force_cg = env("CB_TMA_CG");
    const char* force_bn = env("CB_TMA_BN");
    TmaPlan best{};
    best.cg = 1;  // always-valid default: 1-CTA, 64-channel tiles
    best.bn = 64;
    best.m_tiles = ceil_div64(g.npix, TMA_BM);
    best.n_tiles = (g.kpg + 63) / 64;
    double best_cost = 1e300;
    for (int cg : {1, 2}) {  // ties go to single CTAs (no pair sync; measured faster on cfg1)
        if (force_cg && std::atoi(force_cg) != cg) continue;
        for (int bn : {256, 128, 64}) {
            if (force_bn && std::atoi(force_bn) != bn) continue;
            if (cg == 2 && bn < 128) continue;  // pair MMAs need N >= 128 here
            if (!force_bn && bn > 64 && g.kpg <= bn / 2 && !(cg == 2 && bn == 128)) continue;
            const int64_t m_tiles = ceil_div64(g.npix, (int64_t)TMA_BM * cg);
            const int n_tiles = (g.kpg + bn - 1) / bn;
            const int64_t tiles = m_tiles * n_tiles * g.G;
            const int units = sms / cg;
            const double mma = 12.0 * L.num_kb * (bn / 2.0);
            const double bytes = (double)L.num_kb * (2.0 * TMA_BM * 128 + 2.0 * (bn / cg) * 128);
            const double per_tile = std::max(mma, bytes / 40.0) + 2000.0;
            // full waves, then the ragged tail cut into K parts (the fixup ~10k cycles with
            // its pair / cluster overheads): huge reductions on few tiles fill the GPU
            const int parts = tail_split_parts(tiles, units, L.num_kb, bn);
            const double cost = (double)(tiles / units) * per_tile +
                                (tiles % units ? per_tile / parts + (parts > 1 ? 10000.0 : 0.0) : 0.0);
            if (cost < best_cost * 0.97) {
                best_cost = cost;
                best.cg = cg;
                best.bn = bn;
                best.m_tiles = m_tiles;
                best.n_tiles = n_tiles;
            }
        }
    }
    TmaPlan& pl = best;
    const int units = sms / pl.cg;
    const int64_t tiles = pl.m_tiles * pl.n_tiles * g.G;
    // Atomic split-K (bias pre-fill launch + add epilogue) only on request: by default a
    // short grid is filled by the deterministic tail split below (one launch, no atomics).
    pl.splits = 1;
    const char* splitk = env("CB_TMA_SPLITK");
    if (splitk && std::atoi(splitk) == 1 && tiles < units && L.num_kb >= 4) {
        int want = (int)((units + tiles - 1) / tiles);
        pl.splits = std::max(1, std::min(want, L.num_kb / 2));
    }
    pl.kb_per_split = (L.num_kb + pl.splits - 1) / pl.splits;
    pl.splits = (L.num_kb + pl.kb_per_split - 1) / pl.kb_per_split;
    pl.total_tiles = tiles * pl.splits;
    const int stage_bytes = 2 * TMA_BM * 128 + 2 * (pl.bn / pl.cg) * 128;
    pl.stages = std::min(6, (232448 - 1280 - 2 * 32 * TMA_BM * 4) / stage_bytes);  // - epilogue stage
    // Tail split-K: when whole tiles leave the last wave partly idle -- or a single short
    // wave leaves clusters idle -- cut each tail tile into S K-parts so the last wave fills
    // more clusters.  Parts keep >= 4 K-blocks when the grid is over-full (the fixup must
    // pay off) and >= 2 on a short grid.  Every item then runs on its own CTA (parts <=
    // units / tail), so an owner never waits on a part queued behind it.
    pl.full_items = pl.total_tiles;
    pl.total_items = pl.total_tiles;
    pl.tail_tiles = 0;
    pl.tail_parts = 1;
    pl.tail_kbp = L.num_kb;
    const char* no_tail = env("CB_TMA_TAIL");
    const int64_t tail = tiles % units;
    if (pl.splits == 1 && tail > 0 && !(no_tail && std::atoi(no_tail) == 0)) {
        int parts = tail_split_parts(tiles, units, L.num_kb, pl.bn);
        if (parts >= 2) {
            pl.tail_kbp = (L.num_kb + parts - 1) / parts;
            parts = (L.num_kb + pl.tail_kbp - 1) / pl.tail_kbp;
            pl.tail_tiles = (int)tail;
            pl.tail_parts = parts;
            pl.full_items = tiles - tail;
            pl.total_items = pl.full_items + tail * parts;
        }
    }
    // One item per cluster at a time: tail parts then all run concurrently (required, an
    // owner spins on its parts).  The grid cap is a diagnostic for untailed plans only.
    pl.grid = (int)std::min<int64_t>(pl.total_items, units) * pl.cg;
    if (const char* gcap = env("CB_TMA_GRID"); gcap && pl.tail_tiles == 0)
        pl.grid = std::max(pl.cg, std::min(pl.grid, std::atoi(gcap) / pl.cg * pl.cg));
    return pl;
}

// Extra workspace of the fused conv beyond the activation split: tail counters + partials.
int64_t tma_tail_workspace_bytes(const Geom& g, const FusedLayout& L) {
    if (!L.tma || g.npix == 0) return 0;
    TmaPlan pl = plan_tma(g, L);
    if (pl.tail_tiles == 0) return 0;
    const int64_t ctr = ((int64_t)pl.tail_tiles * pl.cg * 8 + 255) / 256 * 256;  // [written][done]
    return ctr + (int64_t)pl.tail_tiles * pl.tail_parts * pl.cg * pl.bn * TMA_BM * 4;
}
int tma_tail_counters(const Geom& g, const FusedLayout& L) {
    if (!L.tma || g.npix == 0) return 0;
    TmaPlan pl = plan_tma(g, L);
    return 2 * pl.tail_tiles * pl.cg;
}

int tma_plan_query(const Geom& g, bool bf16, cb_tile_plan* out) {
    FusedLayout L = fused_layout(g, bf16);
    TmaPlan pl = plan_tma(g, L);
    out->variant = bf16 ? CB_VARIANT_TC3XBF16 : CB_VARIANT_TC3XTF32;
    out->block_m = TMA_BM * pl.cg;
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

static int make_w_map(CUtensorMap* m, bool bf16, const void* w, int rows, int kw_pad, int box_rows) {
    auto fn = tiled_encode_fn();
    if (!fn) return fail(CB_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    if (reinterpret_cast<uintptr_t>(w) & 15)
        return fail(CB_ERR_MISALIGNED, "packed weights must be 16-byte aligned");
    const int eb = bf16 ? 2 : 4;
    cuuint64_t dims[2] = {(cuuint64_t)kw_pad, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)kw_pad * eb};
    cuuint32_t box[2] = {(cuuint32_t)(128 / eb), (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(m, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                    const_cast<void*>(w), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        return fail(CB_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
    return CB_OK;
}

template <int BN, int STAGES, bool BF16, int CG>
static int launch_tma_cfg(const TmaParams& prm, int grid, const void* ahi, const void* alo,
                          const void* whi, const void* wlo, cudaStream_t st) {
    using Cfg = TmaCfg<BN, STAGES, BF16, CG>;
    auto kern = conv_tma_kernel<BN, STAGES, BF16, CG>;
    static std::once_flag once;
    static cudaError_t attr_err = cudaSuccess;
    std::call_once(once, [&] {
        attr_err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        Cfg::SMEM_BYTES);
    });
    if (attr_err != cudaSuccess)
        return fail(CB_ERR_CUDA, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(attr_err));
    CUtensorMap mah, mal, mwh, mwl, my{};
    int rc;
    if ((rc = make_act_map(&mah, BF16, prm.g, prm.L, ahi))) return rc;
    if ((rc = make_act_map(&mal, BF16, prm.g, prm.L, alo))) return rc;
    if ((rc = make_w_map(&mwh, BF16, whi, prm.g.K, prm.L.kw_pad, Cfg::B_ROWS))) return rc;
    if ((rc = make_w_map(&mwl, BF16, wlo, prm.g.K, prm.L.kw_pad, Cfg::B_ROWS))) return rc;
    if (prm.tma_store) {  // y as {PQ, K, N}, boxes of 128 pixels x 32 channels
        auto fn = tiled_encode_fn();
        cuuint64_t dims[3] = {(cuuint64_t)prm.g.PQ, (cuuint64_t)prm.g.K, (cuuint64_t)prm.g.N};
        cuuint64_t strides[2] = {(cuuint64_t)prm.g.PQ * 4, (cuuint64_t)prm.g.K * prm.g.PQ * 4};
        cuuint32_t box[3] = {(cuuint32_t)TMA_BM, 32, 1};
        cuuint32_t es[3] = {1, 1, 1};
        CUresult r = fn(&my, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, prm.out, dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS)
            return fail(CB_ERR_CUDA, "cuTensorMapEncodeTiled (output) failed: " + std::to_string((int)r));
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(TMA_THREADS);
    cfg.dynamicSmemBytes = Cfg::SMEM_BYTES;
    cfg.stream = st;
    // Tail split-K parts wait on each other across clusters, so every CTA of the grid must
    // be resident at once.  The grid is at most one cluster per co-resident slot of an idle
    // GPU (checked here once per configuration against the occupancy API); a launch that
    // could not be co-resident drops the tail split instead of risking a spin that never
    // ends.  Other kernels running concurrently on other streams can still hold SMs: see
    // the contract in convb200.h (cb_conv_fused_packed).
    if (prm.tail_tiles > 0) {
        static std::once_flag occ_once;
        static int max_units = 0;
        std::call_once(occ_once, [&] {
            if (CG == 2) {
                cudaLaunchConfig_t oc{};
                oc.gridDim = dim3((unsigned)(2 * sm_count()));
                oc.blockDim = dim3(TMA_THREADS);
                oc.dynamicSmemBytes = Cfg::SMEM_BYTES;
                cudaLaunchAttribute ca;
                ca.id = cudaLaunchAttributeClusterDimension;
                ca.val.clusterDim.x = 2;
                ca.val.clusterDim.y = 1;
                ca.val.clusterDim.z = 1;
                oc.attrs = &ca;
                oc.numAttrs = 1;
                if (cudaOccupancyMaxActiveClusters(&max_units, kern, &oc) != cudaSuccess) max_units = 0;
            } else {
                int per_sm = 0;
                if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, TMA_THREADS,
                                                                  Cfg::SMEM_BYTES) != cudaSuccess)
                    per_sm = 0;
                max_units = per_sm * sm_count();
            }
            cudaGetLastError();
        });
        if (grid / CG > max_units)
            return fail(CB_ERR_UNSUPPORTED,
                        "conv_tma: tail split-K grid of " + std::to_string(grid / CG) +
                            " clusters exceeds the " + std::to_string(max_units) +
                            " co-resident clusters this device reports");
    }
    cudaLaunchAttribute attr[2];
    // programmatic dependent launch: the prologue (barriers, TMEM, descriptor prefetch)
    // overlaps the tail of the preceding kernel (K0); griddepcontrol.wait guards the inputs
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = env("CB_NO_PDL") ? 0 : 1;
    // cluster dimension only for CTA pairs (a 1-CTA cluster launch measured ~12% slower on
    // the stepwise GEMM)
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = CG;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = CG == 2 ? 2 : 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, prm, mah, mal, mwh, mwl, my);
    if (e != cudaSuccess) return fail(CB_ERR_CUDA, std::string("conv_tma launch: ") + cudaGetErrorString(e));
    return check_launch("conv_tma_kernel");
}

int launch_fill_bias(int64_t images, int K, int PQ, const float* bias, float* y, cudaStream_t st);

// Diagnostics only (CB_TMA_TRACE set): a library-owned stamp buffer, [cta][TRACE_SLOTS]
// globaltimer values of the latest launch, read back with cb_debug_trace().
static unsigned long long* g_trace = nullptr;
static int g_trace_ctas = 0;
unsigned long long* debug_trace_buffer(int ctas, cudaStream_t st) {
    if (!kTrace) return nullptr;  // product build: no stamps, no buffer
    const size_t n = (size_t)1024 * TRACE_SLOTS;
    if (!g_trace && cudaMalloc(&g_trace, n * sizeof(unsigned long long)) != cudaSuccess)
        g_trace = nullptr;
    if (g_trace) cudaMemsetAsync(g_trace, 0, n * sizeof(unsigned long long), st);
    g_trace_ctas = std::min(ctas, 1024);
    return g_trace;
}
int debug_trace_copy(unsigned long long* host, int max_ctas, int* slots) {
    *slots = TRACE_SLOTS;
    if (!g_trace) return 0;
    cudaDeviceSynchronize();
    const int n = std::min(max_ctas, g_trace_ctas);
    cudaMemcpy(host, g_trace, (size_t)n * TRACE_SLOTS * sizeof(unsigned long long),
               cudaMemcpyDeviceToHost);
    return n;
}

// The TMA conv proper (K6), activations already split into the NHWC workspace.
int launch_conv_tma(bool bf16, const Geom& g, const FusedLayout& L, const void* act_hi,
                    const void* act_lo, const void* w_hi, const void* w_lo, const float* bias,
                    float* y, void* tail_ws, cudaStream_t st) {
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
    prm.full_items = pl.full_items;
    prm.total_items = pl.total_items;
    prm.tail_last = env("CB_TMA_TAIL_LAST") ? 1 : 0;
    prm.tail_tiles = pl.tail_tiles;
    prm.tail_parts = pl.tail_parts;
    prm.tail_kbp = pl.tail_kbp;
    if (pl.tail_tiles > 0) {
        if (!tail_ws) return fail(CB_ERR_WORKSPACE, "tail split-K needs workspace");
        const int64_t ctr = ((int64_t)pl.tail_tiles * pl.cg * 8 + 255) / 256 * 256;
        prm.counters = static_cast<int*>(tail_ws);
        prm.partials = reinterpret_cast<float*>(static_cast<uint8_t*>(tail_ws) + ctr);
    }
    prm.add_mode = 0;
    if (const char* dbg = env("CB_TMA_DEBUG")) prm.debug = std::atoi(dbg);
    // Optional TMA-store epilogue (CB_TMA_TSTORE) and bulk-copy tail partials
    // (CB_TMA_BULK_PARTS): measured equal or slower than the direct stores on cfg4 and on
    // output-heavy sweep ops (two epilogue barriers per chunk; tiles crossing images fall
    // back to direct stores anyway), so both are off by default.
    prm.tma_store = (g.PQ % 4 == 0) && (g.G == 1 || g.kpg % 32 == 0) &&
                    (reinterpret_cast<uintptr_t>(y) & 15) == 0 && env("CB_TMA_TSTORE");
    prm.bulk_parts = env("CB_TMA_BULK_PARTS") ? 1 : 0;
    prm.out_al16 = (reinterpret_cast<uintptr_t>(y) & 15) == 0 ? 1 : 0;
    prm.range_kb = std::max(1, promote_k(bf16) / (128 / L.eb));
    if (env("CB_TMA_TRACE")) prm.trace = debug_trace_buffer(pl.grid, st);
    if (pl.splits > 1) {
        int rc = launch_fill_bias(g.N, g.K, g.PQ, bias, y, st);
        if (rc) return rc;
        prm.add_mode = 1;
        prm.tma_store = 0;
    }
#define CB_TMA_CASE(CG_, BN_, ST_)                                                               \
    if (pl.cg == CG_ && pl.bn == BN_ && pl.stages == ST_)                                         \
        return bf16 ? launch_tma_cfg<BN_, ST_, true, CG_>(prm, pl.grid, act_hi, act_lo, w_hi, w_lo, st) \
                    : launch_tma_cfg<BN_, ST_, false, CG_>(prm, pl.grid, act_hi, act_lo, w_hi, w_lo, st);
    // stage counts = floor(227 KB / stage bytes), see plan_tma
    CB_TMA_CASE(1, 256, 2)
    CB_TMA_CASE(1, 128, 3)
    CB_TMA_CASE(1, 64, 4)
    CB_TMA_CASE(2, 256, 3)
    CB_TMA_CASE(2, 128, 4)
#undef CB_TMA_CASE
    return fail(CB_ERR_UNSUPPORTED, "no TMA tile configuration for cg=" + std::to_string(pl.cg) +
                                        " bn=" + std::to_string(pl.bn) +
                                        " stages=" + std::to_string(pl.stages));
}

}  // namespace cb
