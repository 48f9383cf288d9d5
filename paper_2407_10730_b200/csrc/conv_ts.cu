// conv_ts.cu -- K7: direct tcgen05 convolution for few-channel layers (short reductions,
// C*R*S <= ~200, e.g. the 3-channel 7x7 stem of config 3).
//
// The TMA path (K0 + K6) pads every tap of a 3-channel conv to a 16-byte chunk and round-
// trips a re-laid-out copy of the input through HBM; with N = 64 output channels its
// shared-memory-operand MMAs are bound by the A-operand reads.  Here instead:
//
//   * the TMA warp stages the zero-padded fp32 input rows one 128-pixel tile needs
//     ([C][rows][W + 2*pw] box of the NCHW tensor, out-of-range rows/cols zero-filled by
//     the TMA unit) into a ring of smem windows, and loads the split weights once;
//   * the producer warps (CB_TS_KPARTS per TMEM lane quadrant, default one: the kernel is
//     bound by shared-memory bandwidth, more producers only add per-tile overhead) build
//     the tile's A operand -- pixel row m, reduction k in the plan's layout (OIHW order,
//     padded tap pairs, or the mixed pairs + singles layout of cb_common.cuh) -- from
//     the window, split every value into bf16 (hi, lo) and write both halves straight into
//     TMEM with tcgen05.st (no smem A tile, no activation pre-pass, no workspace);
//   * the MMA warp issues, per 16-wide K step, A_lo*B_hi, A_hi*B_lo, A_hi*B_hi as
//     tcgen05.mma kind::f16 with A read from TMEM and B (weights, K-major SW128) from smem;
//   * four epilogue warps drain the double-buffered TMEM accumulator into NCHW (+bias).
//
// The 3xTF32 split (compile-time layouts) keeps tf32 words in TMEM instead of bf16 pairs --
// hi is the value itself, lo = v - trunc_tf32(v), no conversions -- and issues kind::tf32
// MMAs of 8 reduction elements; when only one whole-K A buffer fits, it is used as two
// half-K buffers so the build of one half overlaps the MMAs of the other.
//
// Tiles are 128 consecutive output pixels of one image; the persistent grid walks them.
// HBM traffic is the algorithmic minimum: x read once (the window re-reads hit L2), y
// written once, the weights once per CTA.
#include <cudaTypedefs.h>

#include <mutex>
#include <set>

#include "cb_common.cuh"
#include "sm100_ptx.cuh"

namespace cb {

constexpr int TS_BM = 128;
#ifndef CB_TS_KPARTS
#define CB_TS_KPARTS 1
#endif
#ifndef CB_TS_DEPTH
#define CB_TS_DEPTH 3  // 8-element groups of window loads in flight ahead of the split
#endif
#ifndef CB_TS_STW
#define CB_TS_STW 1  // 8-element groups per tcgen05.st (1, 2 or 4: .x4 / .x8 / .x16)
#endif
constexpr int TS_PROD_WARPS = 4 * CB_TS_KPARTS;  // CB_TS_KPARTS per TMEM lane quadrant
constexpr int TS_EPI_WARP0 = TS_PROD_WARPS;
constexpr int TS_TMA_WARP = TS_PROD_WARPS + 4;
constexpr int TS_MMA_WARP = TS_PROD_WARPS + 5;
constexpr int TS_THREADS = (TS_PROD_WARPS + 6) * 32;
constexpr int TS_TMEM_COLS = 512;

struct TsParams {
    Geom g;
    const float* bias;
    float* out;
    int kp;             // reduction padded to 32 (A columns per half: kp / 2 for bf16 pairs,
                        // kp for tf32 words)
    int nab;            // A buffers in TMEM: 2, or 1 when only one fits (tf32)
    int acols;          // TMEM columns of one A buffer (hi + lo halves)
    int ksteps_real;    // MMA K steps that hold reduction elements (the rest of kp is zero padding)
    int khalves;        // 2: the single tf32 A buffer is used as two half-K buffers (a ring over
                        // (tile, K half): the build of one half overlaps the MMAs of the other)
    int n_pad;          // output channels padded to 16 (MMA N)
    int kb_w;           // split weight row length (multiple of 64)
    int tiles_per_img;  // ceil(PQ / (128 * CG)): tiles of one CTA (CG = 1) or pair (CG = 2)
    int64_t total_tiles;
    int box_rows, box_w;    // staging window: input rows x padded row width
    int x0;                 // window column 0 = input column -x0 (x0 = pw rounded up to 4)
    uint32_t stage_bytes;   // C * box_rows * box_w * 4 (TMA transaction bytes)
    uint32_t stage_stride;  // stage_bytes rounded to 1 KB (buffer pitch)
    int nwin;               // staging windows in the ring (2..4): the window TMA of tile i +
                            // nwin - 1 is in flight while tile i is built (its L2 latency,
                            // ~2.6k cycles on cfg3, exceeds one tile's A build)
    uint32_t w_half_bytes;  // (n_pad / CG) * kb_w * 2: this CTA's weight rows, one half
    int w_rows;             // n_pad / CG
    int debug;              // diagnostics (CB_TS_DEBUG): 1 no MMA, 2 no tcgen05.st, 4 no input TMA
    int tma_store;          // 1: epilogue stages 32-channel chunks in smem, TMA stores them
    float inv_q;            // 1 / Q (pixel -> output row without an integer division)
    int fixed;              // CB_TS_FIXED_LIST id of a compile-time producer, 0: generic
    // pair mode (fixed producers, even horizontal stride, odd S): the reduction is laid out
    // k = (c*R + r)*(S+1) + s' with one zero-weight pad tap per (c, r) row -- at s' = 0 when
    // pf = 1, at s' = S otherwise -- so each k pair (s', s'+1) is one 8-byte aligned LDS.64
    // of two adjacent window columns (the A build is bound by the LDS instruction rate)
    int pair;
    int pf;
    unsigned long long* trace;  // diagnostics (CB_TS_TRACE): clock64 stamps of CTAs 0..3
};

// Persistent tile walk without 64-bit divisions: tile t = n * tiles_per_img + ti, advanced
// by gridDim.x = step_n * tiles_per_img + step_ti.
struct TileWalk {
    int t, n, ti, step_n, step_ti, units;
    __device__ __forceinline__ TileWalk(const struct TsParams& p, int unit, int nunits);
    __device__ __forceinline__ void next(const struct TsParams& p);
};

// trace layout: [cta < 4][event < 16][local tile < 512]
__device__ __forceinline__ void ts_stamp(const TsParams& p, int e, int i) {
    if (kTrace && p.trace && blockIdx.x < 4 && i < 512) p.trace[blockIdx.x * 8192 + e * 512 + i] = clock64();
}

__device__ __forceinline__ TileWalk::TileWalk(const TsParams& p, int unit, int nunits) {
    t = unit;
    units = nunits;
    n = t / p.tiles_per_img;
    ti = t - n * p.tiles_per_img;
    step_n = nunits / p.tiles_per_img;
    step_ti = nunits - step_n * p.tiles_per_img;
}
__device__ __forceinline__ void TileWalk::next(const TsParams& p) {
    t += units;
    n += step_n;
    ti += step_ti;
    if (ti >= p.tiles_per_img) {
        ti -= p.tiles_per_img;
        ++n;
    }
}
// v / Q for 0 <= v < 2^21: (v + 0.5) / Q stays >= 0.5 / Q away from an integer, far above
// the float rounding error
__device__ __forceinline__ int div_q(int v, const TsParams& p) {
    return __float2int_rz(((float)v + 0.5f) * p.inv_q);
}

__device__ __forceinline__ float lds_f32(uint32_t a) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts_f32(uint32_t a, float v) {
    asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"(v) : "memory");
}
__device__ __forceinline__ int4 lds_v4(uint32_t a) {
    int4 v;
    asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "r"(a));
    return v;
}

// two fp32 -> packed bf16 pair (round to nearest even), element `lo_elem` in bits 0..15
__device__ __forceinline__ uint32_t bf16x2_rn(float lo_elem, float hi_elem) {
    uint32_t d;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(hi_elem), "f"(lo_elem));
    return d;
}

// (hi, lo) bf16 pair words of two fp32 values: hi = (bf16(v0), bf16(v1)), lo = the rounded
// residuals, element v0 in bits 0..15
__device__ __forceinline__ void split_pair(float v0, float v1, uint32_t& hi, uint32_t& lo) {
    hi = bf16x2_rn(v0, v1);
    lo = bf16x2_rn(v0 - __uint_as_float(hi << 16), v1 - __uint_as_float(hi & 0xffff0000u));
}

// One group of 8 reduction elements (4 value pairs) split and written to the A buffer: bf16
// halves as 4 + 4 packed words (group g at column 4g), tf32 halves as 8 + 8 words (column 8g).
template <bool BF16>
__device__ __forceinline__ void split_store_group(const float (&u)[8], uint32_t a_hi, uint32_t a_lo, int g) {
    if constexpr (BF16) {
        uint32_t hv[4], lv[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) split_pair(u[2 * e], u[2 * e + 1], hv[e], lv[e]);
        ptx::tmem_st_32x32b_groups(a_hi + g * 4, hv, 1);
        ptx::tmem_st_32x32b_groups(a_lo + g * 4, lv, 1);
    } else {
        uint32_t hv[8], lv[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            // kind::tf32 reads the top 19 bits of an operand word, so the hi half is the
            // value itself and lo = v - trunc_tf32(v) is exact (<= 13 significant bits, read
            // to 11: 2^-21 |v|, below the dropped lo * lo term).  No cvt.rna.tf32 -- those
            // conversions made the tf32 build 2.7x the bf16 one (2680 vs 980 cycles a tile).
            const uint32_t bits = __float_as_uint(u[e]);
            hv[e] = bits;
            lv[e] = __float_as_uint(u[e] - __uint_as_float(bits & 0xffffe000u));
        }
        ptx::tmem_st_32x32b_groups(a_hi + g * 8, hv, 2);
        ptx::tmem_st_32x32b_groups(a_lo + g * 8, lv, 2);
    }
}

// A producer with the reduction layout fixed at compile time (C, R, S, unit horizontal
// dilation): groups [G0, G1) of 8 reduction elements k = (c, r, s), each element one LDS at
// xs + c * cstride + r * rstride + 4 s (the (c, r) row offsets are loop-invariant, the tap an
// immediate) -- no offset table, no per-element address arithmetic.  Elements past C*R*S
// are written as zeros.
template <int C, int R, int S>
__device__ __forceinline__ void load_pair(int k, uint32_t xs, uint32_t xa, uint32_t xb, uint32_t cstride,
                                          uint32_t rstride, bool swap, float& v0, float& v1) {
    constexpr int KD = C * R * S;
    const int c = k / (R * S), rs = k % (R * S);
    if (k + 1 < KD && rs % S + 1 < S) {  // taps (s, s + 1) of one (c, r) row
        const uint32_t off = c * cstride + (rs / S) * rstride + 4 * (rs % S);
        v0 = lds_f32(xa + off);  // lanes 16..31 (swap): the second tap
        v1 = lds_f32(xb + off);
        if (swap) {
            const float t = v0;
            v0 = v1;
            v1 = t;
        }
    } else {
        v0 = k < KD ? lds_f32(xs + c * cstride + (rs / S) * rstride + 4 * (rs % S)) : 0.f;
        const int c1 = (k + 1) / (R * S), rs1 = (k + 1) % (R * S);
        v1 = k + 1 < KD ? lds_f32(xs + c1 * cstride + (rs1 / S) * rstride + 4 * (rs1 % S)) : 0.f;
    }
}

// Groups [G0, G1) of 8 elements, software-pipelined: the loads of group g + D are issued
// before group g is split and stored (the volatile LDS / tcgen05.st asm statements keep
// their source order, so without this every group would wait out a full LDS latency).
template <int C, int R, int S, int G0, int G1, bool BF16 = true>
__device__ __forceinline__ void build_fixed(uint32_t xs, uint32_t cstride, uint32_t rstride,
                                            uint32_t a_hi, uint32_t a_lo, bool swap) {
    constexpr int NG = G1 - G0, D = CB_TS_DEPTH;
    // swap (even horizontal stride): lanes 16..31 load the second tap of an adjacent pair
    // first, so the warp's 32 addresses (2 words apart per pixel) cover all 32 banks
    const uint32_t xa = xs + (swap ? 4u : 0u), xb = xs + (swap ? 0u : 4u);
    constexpr int W = CB_TS_STW;
    float v[D + 1][8];
    uint32_t hv[4 * W], lv[4 * W];
#pragma unroll
    for (int step = 0; step < NG + D; ++step) {
        if (step < NG) {
#pragma unroll
            for (int e = 0; e < 8; e += 2)
                load_pair<C, R, S>((G0 + step) * 8 + e, xs, xa, xb, cstride, rstride, swap,
                                   v[step % (D + 1)][e], v[step % (D + 1)][e + 1]);
        }
        if (step >= D) {
            const int gi = step - D;
            const float* u = v[gi % (D + 1)];
            if constexpr (!BF16) {
                split_store_group<false>(v[gi % (D + 1)], a_hi, a_lo, G0 + gi);
                continue;
            }
            const int slot = gi % W;
#pragma unroll
            for (int e = 0; e < 4; ++e) split_pair(u[2 * e], u[2 * e + 1], hv[slot * 4 + e], lv[slot * 4 + e]);
            if (slot == W - 1 || gi == NG - 1) {  // W groups (or the rest) per tcgen05.st
                ptx::tmem_st_32x32b_groups(a_hi + (G0 + gi - slot) * 4, hv, slot + 1);
                ptx::tmem_st_32x32b_groups(a_lo + (G0 + gi - slot) * 4, lv, slot + 1);
            }
        }
    }
}

// Pair-mode producer: groups [G0, G1) of 8 elements of the padded layout (S' = S + 1 taps a
// row, even), each pair one LDS.64 at xs_pair + row offset + 8 * (s' / 2).
template <int C, int R, int S, int G0, int G1>
__device__ __forceinline__ void build_pairs(uint32_t xs_pair, uint32_t cstride, uint32_t rstride,
                                            uint32_t a_hi, uint32_t a_lo) {
    constexpr int SP = S + 1, KD = C * R * SP, NG = G1 - G0, D = CB_TS_DEPTH;
    constexpr int W = CB_TS_STW;
    float2 v[D + 1][4];
    uint32_t hv[4 * W], lv[4 * W];
#pragma unroll
    for (int step = 0; step < NG + D; ++step) {
        if (step < NG) {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int k = (G0 + step) * 8 + 2 * e;
                if (k < KD) {
                    const int cr = k / SP, sp = k % SP;
                    const uint32_t a = xs_pair + (cr / R) * cstride + (cr % R) * rstride + 4 * sp;
                    asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];"
                                 : "=f"(v[step % (D + 1)][e].x), "=f"(v[step % (D + 1)][e].y)
                                 : "r"(a));
                } else {
                    v[step % (D + 1)][e] = make_float2(0.f, 0.f);
                }
            }
        }
        if (step >= D) {
            const int gi = step - D;
            const int slot = gi % W;
#pragma unroll
            for (int e = 0; e < 4; ++e)
                split_pair(v[gi % (D + 1)][e].x, v[gi % (D + 1)][e].y, hv[slot * 4 + e], lv[slot * 4 + e]);
            if (slot == W - 1 || gi == NG - 1) {  // W groups (or the rest) per tcgen05.st
                ptx::tmem_st_32x32b_groups(a_hi + (G0 + gi - slot) * 4, hv, slot + 1);
                ptx::tmem_st_32x32b_groups(a_lo + (G0 + gi - slot) * 4, lv, slot + 1);
            }
        }
    }
}

// Mixed-layout producer (cb_common.cuh: mixed_map): groups [G0, G1) of 8 elements; a k pair
// inside a row's pair region is one LDS.64, the pair of two rows' single taps two LDS.32.
template <int C, int R, int S, int PF, int G0, int G1, bool BF16 = true>
__device__ __forceinline__ void build_mixed(uint32_t xs, uint32_t cstride, uint32_t rstride,
                                            uint32_t a_hi, uint32_t a_lo) {
    constexpr int NR = C * R, NG = G1 - G0, D = CB_TS_DEPTH;
    constexpr int W = CB_TS_STW;
    float2 v[D + 1][4];
    uint32_t hv[4 * W], lv[4 * W];
#pragma unroll
    for (int step = 0; step < NG + D; ++step) {
        if (step < NG) {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int k = (G0 + step) * 8 + 2 * e;
                const MixedTap t0 = mixed_map(k, NR, S, PF), t1 = mixed_map(k + 1, NR, S, PF);
                float2& d = v[step % (D + 1)][e];
                if (t0.cr >= 0 && t1.cr == t0.cr && t1.s == t0.s + 1) {  // aligned tap pair
                    const uint32_t a = xs + (t0.cr / R) * cstride + (t0.cr % R) * rstride + 4 * t0.s;
                    asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(d.x), "=f"(d.y) : "r"(a));
                } else {
                    d.x = t0.cr >= 0 ? lds_f32(xs + (t0.cr / R) * cstride + (t0.cr % R) * rstride + 4 * t0.s) : 0.f;
                    d.y = t1.cr >= 0 ? lds_f32(xs + (t1.cr / R) * cstride + (t1.cr % R) * rstride + 4 * t1.s) : 0.f;
                }
            }
        }
        if (step >= D) {
            const int gi = step - D;
            if constexpr (!BF16) {
                const float2* q = v[gi % (D + 1)];
                const float u[8] = {q[0].x, q[0].y, q[1].x, q[1].y, q[2].x, q[2].y, q[3].x, q[3].y};
                split_store_group<false>(u, a_hi, a_lo, G0 + gi);
                continue;
            }
            const int slot = gi % W;
#pragma unroll
            for (int e = 0; e < 4; ++e)
                split_pair(v[gi % (D + 1)][e].x, v[gi % (D + 1)][e].y, hv[slot * 4 + e], lv[slot * 4 + e]);
            if (slot == W - 1 || gi == NG - 1) {  // W groups (or the rest) per tcgen05.st
                ptx::tmem_st_32x32b_groups(a_hi + (G0 + gi - slot) * 4, hv, slot + 1);
                ptx::tmem_st_32x32b_groups(a_lo + (G0 + gi - slot) * 4, lv, slot + 1);
            }
        }
    }
}

template <int C, int R, int S, int PF, bool BF16 = true>
__device__ __forceinline__ void build_mixed_part(int kpart, uint32_t xs, uint32_t cstride,
                                                 uint32_t rstride, uint32_t a_hi, uint32_t a_lo) {
    constexpr int G = (mixed_kdim(C * R, S) + 7) / 8, P = CB_TS_KPARTS;
    if (kpart == 0)
        build_mixed<C, R, S, PF, 0, G * 1 / P, BF16>(xs, cstride, rstride, a_hi, a_lo);
    else if (kpart == 1 && P > 1)
        build_mixed<C, R, S, PF, G * 1 / P, G * 2 / P, BF16>(xs, cstride, rstride, a_hi, a_lo);
    else if (kpart == 2 && P > 2)
        build_mixed<C, R, S, PF, G * 2 / P, G * 3 / P, BF16>(xs, cstride, rstride, a_hi, a_lo);
    else if (P > 3)
        build_mixed<C, R, S, PF, G * 3 / P, G, BF16>(xs, cstride, rstride, a_hi, a_lo);
}

template <int C, int R, int S>
__device__ __forceinline__ void build_pairs_part(int kpart, uint32_t xs_pair, uint32_t cstride,
                                                 uint32_t rstride, uint32_t a_hi, uint32_t a_lo) {
    constexpr int G = (C * R * (S + 1) + 7) / 8, P = CB_TS_KPARTS;
    if (kpart == 0)
        build_pairs<C, R, S, 0, G * 1 / P>(xs_pair, cstride, rstride, a_hi, a_lo);
    else if (kpart == 1 && P > 1)
        build_pairs<C, R, S, G * 1 / P, G * 2 / P>(xs_pair, cstride, rstride, a_hi, a_lo);
    else if (kpart == 2 && P > 2)
        build_pairs<C, R, S, G * 2 / P, G * 3 / P>(xs_pair, cstride, rstride, a_hi, a_lo);
    else if (P > 3)
        build_pairs<C, R, S, G * 3 / P, G>(xs_pair, cstride, rstride, a_hi, a_lo);
}

// the producer warps of a lane quadrant take contiguous shares of the 8-element groups
template <int C, int R, int S, bool BF16 = true>
__device__ __forceinline__ void build_fixed_part(int kpart, uint32_t xs, uint32_t cstride,
                                                 uint32_t rstride, uint32_t a_hi, uint32_t a_lo,
                                                 bool swap) {
    constexpr int G = (C * R * S + 7) / 8, P = CB_TS_KPARTS;
    if (kpart == 0)
        build_fixed<C, R, S, 0, G * 1 / P, BF16>(xs, cstride, rstride, a_hi, a_lo, swap);
    else if (kpart == 1 && P > 1)
        build_fixed<C, R, S, G * 1 / P, G * 2 / P, BF16>(xs, cstride, rstride, a_hi, a_lo, swap);
    else if (kpart == 2 && P > 2)
        build_fixed<C, R, S, G * 2 / P, G * 3 / P, BF16>(xs, cstride, rstride, a_hi, a_lo, swap);
    else if (P > 3)
        build_fixed<C, R, S, G * 3 / P, G, BF16>(xs, cstride, rstride, a_hi, a_lo, swap);
}

// compile-time reduction layouts (TsParams::fixed): 0 = generic offset-table producer
#define CB_TS_FIXED_LIST(X) X(1, 3, 7, 7) X(2, 3, 3, 3) X(3, 3, 5, 5) X(4, 4, 3, 3) X(5, 4, 7, 7)
template <int FX>
struct TsLayout {
    static constexpr int C = 0, R = 0, S = 0;
};
#define CB_TS_LAYOUT(id, c, r, s)          \
    template <>                            \
    struct TsLayout<id> {                  \
        static constexpr int C = c, R = r, S = s; \
    };
CB_TS_FIXED_LIST(CB_TS_LAYOUT)
#undef CB_TS_LAYOUT

// One instantiation per (CTA group, compile-time layout FX, pair mode): each kernel holds
// only its own unrolled producer -- with all layouts in one kernel the ncu profile showed
// 12% of warp stalls as no_instructions (instruction-cache misses).
// MODE: 0 plain, 1 padded pairs, 2 / 3 mixed layout with pf = 0 / 1.  BF16 = false: the 3xTF32
// split (tf32 words in TMEM, kind::tf32 MMAs of 8 reduction elements; compile-time layouts,
// single CTAs, MODE 0 / 2 / 3 only).
template <int CG, int FX, int MODE, bool BF16 = true>
__global__ void __launch_bounds__(TS_THREADS, 1)
conv_ts_kernel(const __grid_constant__ TsParams p, const __grid_constant__ CUtensorMap tm_x,
               const __grid_constant__ CUtensorMap tm_whi, const __grid_constant__ CUtensorMap tm_wlo,
               const __grid_constant__ CUtensorMap tm_y) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    uint8_t* w_hi = smem;
    uint8_t* w_lo = smem + p.w_half_bytes;
    float* stage0 = reinterpret_cast<float*>(smem + 2 * p.w_half_bytes);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 2 * p.w_half_bytes + p.nwin * p.stage_stride);
    uint64_t* w_full = bars;            // 1
    uint64_t* s_full = bars + 1;        // 4: staging window landed
    uint64_t* s_empty = bars + 5;       // 4: producers done with the window
    uint64_t* a_full = bars + 9;        // 2: A buffer written
    uint64_t* a_empty = bars + 11;      // 2: MMAs done reading the A buffer
    uint64_t* acc_full = bars + 13;     // 2: accumulator ready
    uint64_t* acc_empty = bars + 15;    // 2: epilogue drained the accumulator
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 17);
    // epilogue staging: 2 x [32 channels][128 pixels] fp32 (after the barriers, 1 KB aligned)
    float* ostage = reinterpret_cast<float*>(smem + 2 * p.w_half_bytes + p.nwin * p.stage_stride + 1024);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const Geom& g = p.g;
    // CTA pair (CG = 2): each CTA stages its own window, builds its own 128 pixel rows of A
    // in its own TMEM and holds half of the weight rows; the leader (rank 0) issues M = 256
    // MMAs over both, and the commits multicast to both CTAs' barriers.
    const uint32_t rank = CG == 2 ? ptx::cluster_ctarank() : 0;
    const int unit0 = (int)blockIdx.x / CG, nunits = (int)gridDim.x / CG;
    const int col_a0 = 2 * p.n_pad;  // TMEM: [acc0 | acc1 | A0 (hi, lo) | A1 (hi, lo)]
    const int half_cols = (BF16 || p.khalves == 2) ? p.kp / 2 : p.kp;

    if (threadIdx.x == 0) {
        ptx::mbar_init(w_full, 1);
        for (int b = 0; b < p.nwin; ++b) {
            ptx::mbar_init(&s_full[b], 1);
            ptx::mbar_init(&s_empty[b], TS_PROD_WARPS);
        }
        for (int b = 0; b < 2; ++b) {
            ptx::mbar_init(&a_full[b], CG * TS_PROD_WARPS);
            ptx::mbar_init(&a_empty[b], 1);
            ptx::mbar_init(&acc_full[b], 1);
            ptx::mbar_init(&acc_empty[b], CG * 4);  // one arriving lane per epilogue warp
        }
        ptx::fence_mbar_init();
    }
    if (warp == TS_TMA_WARP && lane == 0) {
        ptx::tma_prefetch_desc(&tm_x);
        ptx::tma_prefetch_desc(&tm_whi);
        ptx::tma_prefetch_desc(&tm_wlo);
    }
    if (warp == TS_MMA_WARP) {
        if (CG == 2)
            ptx::tmem_alloc_pair(tmem_slot, TS_TMEM_COLS);
        else
            ptx::tmem_alloc(tmem_slot, TS_TMEM_COLS);
    }
    ptx::tc_fence_before();
    if (CG == 2)
        ptx::cluster_sync();
    else
        __syncthreads();
    ptx::tc_fence_after();
    // everything above (barriers, TMEM, descriptor prefetch) touches no global memory: with
    // a programmatic launch it overlaps the stream predecessor's tail
    ptx::grid_dependency_wait();
    // the leader's barriers, addressed from either CTA of a pair
    const uint32_t a_full_l0 = CG == 2 ? ptx::mapa_shared(ptx::smem_u32(&a_full[0]), 0) : 0;
    const uint32_t acc_empty_l0 = CG == 2 ? ptx::mapa_shared(ptx::smem_u32(&acc_empty[0]), 0) : 0;
    const uint32_t tmem_base = *tmem_slot;
    if (threadIdx.x == 0) ts_stamp(p, 15, 0);

    if (warp < TS_PROD_WARPS) {
        // ============================ A producers ======================================
        // koff[k] = window offset of reduction element k = (c, r, s) relative to the pixel's
        // window origin (the same for every pixel); k >= kdim points at a finite value
        // (the matching weight rows are zero).  Per element: one LDS, then the (hi, lo)
        // split with paired bf16x2 conversions -- no predicates in the loop.
        int* koff = reinterpret_cast<int*>(ostage + 2 * 32 * TS_BM);
        for (int k = threadIdx.x; k < p.kp; k += 32 * TS_PROD_WARPS) {
            int o = 0;
            if (k < g.kdim) {
                const int c = k / g.RS, rs = k - (k / g.RS) * g.RS;
                const int r = rs / g.S, s2 = rs - (rs / g.S) * g.S;
                o = (c * p.box_rows + r * g.dh) * p.box_w + s2 * g.dw;
            }
            koff[k] = 4 * o;  // byte offset
        }
        asm volatile("bar.sync 2, %0;" ::"n"(32 * TS_PROD_WARPS) : "memory");
        const int quad = warp & 3, kpart = warp >> 2;
        constexpr int KPARTS = TS_PROD_WARPS / 4;
        const int m = quad * 32 + lane;  // pixel row of the tile == TMEM lane
        const uint32_t lane_addr = tmem_base + ((uint32_t)(quad * 32) << 16);
        const int nchunks = p.kp / 32;
        const bool swap = (g.sw % 2 == 0) && lane >= 16 && !(p.debug & 32);
        // The tile loop is software-pipelined across tiles: the next tile's window origin and
        // the (non-blocking) tests of its two barriers are issued before this tile's
        // tcgen05.st drain, so their latencies (~250-400 cycles a tile when taken in
        // sequence at the top of the loop) overlap the drain and the hand-off.  One lane per
        // warp arrives (after __syncwarp) instead of 32.
        auto window_origin = [&](const TileWalk& tw, int ws) -> uint32_t {
            // this CTA's first pixel; past the image (the second half of a pair's last tile)
            // the window origin stays inside it and nothing is stored
            const int p0 = min(tw.ti * (TS_BM * CG) + (int)rank * TS_BM, g.PQ - 1);
            const int oy_a = div_q(p0, p);
            const int pix = min(p0 + m, g.PQ - 1);  // rows past the image: finite, never stored
            const int oy = div_q(pix, p);
            const int ox = pix - oy * g.Q;
            return ptx::smem_u32(stage0) + ws * p.stage_stride +
                   4u * (uint32_t)((oy - oy_a) * g.sh * p.box_w + ox * g.sw + (p.x0 - g.pw));
        };
        int i = 0;
        int ws = 0;  // staging-window ring slot and phase
        uint32_t wph = 0;
        TileWalk tw(p, unit0, nunits);
        bool have = tw.t < p.total_tiles;
        uint32_t xs = 0;
        if (have) {
            xs = window_origin(tw, ws);
            ptx::mbar_wait(&s_full[ws], wph);
            ptx::mbar_wait(&a_empty[0], 1);
            ptx::tc_fence_after();
        }
        while (have) {
            const bool halves = !BF16 && FX != 0 && KPARTS == 1 && p.khalves == 2;
            const int b = p.nab == 2 ? (i & 1) : halves ? 1 : 0;  // A buffer this iteration hands over last
            if (lane == 0 && (warp == 0 || warp == 8)) ts_stamp(p, warp == 0 ? 2 : 12, i);
            const uint32_t a_hi = lane_addr + col_a0 + b * p.acols;
            const uint32_t a_lo = a_hi + half_cols;
            if constexpr (!BF16 && FX != 0 && KPARTS == 1) {
                if (halves) {
                    const bool build = !(p.debug & 16);
                    // K halves: groups [0, GH) go to buffer 0 and are handed to the MMA warp,
                    // then groups [GH, G) to buffer 1 (each buffer kp columns: hi | lo)
                    using L = TsLayout<FX>;
                    constexpr int KD = MODE >= 2 ? mixed_kdim(L::C * L::R, L::S) : L::C * L::R * L::S;
                    constexpr int KP = (KD + 31) / 32 * 32, G = (KD + 7) / 8, GH = KP / 16;
                    static_assert(G > GH, "the second K half holds at least one group");
                    const uint32_t cstride = 4u * p.box_rows * p.box_w, rstride = 4u * g.dh * p.box_w;
                    const uint32_t base0 = lane_addr + col_a0, base1 = base0 + KP;
                    if (build) {
                        if constexpr (MODE >= 2)
                            build_mixed<L::C, L::R, L::S, MODE - 2, 0, GH, false>(xs, cstride, rstride, base0, base0 + KP / 2);
                        else
                            build_fixed<L::C, L::R, L::S, 0, GH, false>(xs, cstride, rstride, base0, base0 + KP / 2, swap);
                    }
                    ptx::tmem_st_wait();
                    ptx::tc_fence_before();
                    __syncwarp();
                    if (lane == 0) ptx::mbar_arrive(&a_full[0]);
                    ptx::mbar_wait(&a_empty[1], (uint32_t)(i & 1) ^ 1);
                    ptx::tc_fence_after();
                    if (i == 0 && build) {  // columns past the written groups of the second half: zero once
                        const uint32_t z[4] = {0u, 0u, 0u, 0u};
                        for (int c4 = (G - GH) * 8; c4 < KP / 2; c4 += 4) {
                            ptx::tmem_st_32x32b_x4(base1 + c4, z);
                            ptx::tmem_st_32x32b_x4(base1 + KP / 2 + c4, z);
                        }
                    }
                    if (build) {
                        if constexpr (MODE >= 2)
                            build_mixed<L::C, L::R, L::S, MODE - 2, GH, G, false>(xs, cstride, rstride, base1 - GH * 8,
                                                                                  base1 + KP / 2 - GH * 8);
                        else
                            build_fixed<L::C, L::R, L::S, GH, G, false>(xs, cstride, rstride, base1 - GH * 8,
                                                                        base1 + KP / 2 - GH * 8, swap);
                    }
                }
            }
            if (FX != 0 && !(p.debug & 16) && !halves) {
                if (i < p.nab) {  // columns past the written groups: zero once per A buffer
                    const uint32_t z[4] = {0u, 0u, 0u, 0u};
                    const int kd = MODE == 1 ? g.C * g.R * (g.S + 1) : MODE >= 2 ? mixed_kdim(g.C * g.R, g.S) : g.kdim;
                    for (int c4 = ((kd + 7) / 8) * (BF16 ? 4 : 8) + kpart * 4; c4 < half_cols; c4 += 4 * KPARTS) {
                        ptx::tmem_st_32x32b_x4(a_hi + c4, z);
                        ptx::tmem_st_32x32b_x4(a_lo + c4, z);
                    }
                }
                const uint32_t cstride = 4u * p.box_rows * p.box_w, rstride = 4u * g.dh * p.box_w;
                using L = TsLayout<FX>;
                if constexpr (FX != 0 && MODE >= 2 && L::S % 2 == 1) {
                    build_mixed_part<L::C, L::R, L::S, MODE - 2, BF16>(kpart, xs, cstride, rstride, a_hi, a_lo);
                } else if constexpr (FX != 0 && MODE == 1 && L::S % 2 == 1) {
                    const uint32_t xs_pair = xs - 4u * p.pf;  // 8-byte aligned (plan_ts)
                    build_pairs_part<L::C, L::R, L::S>(kpart, xs_pair, cstride, rstride, a_hi, a_lo);
                } else if constexpr (FX != 0 && MODE == 0) {
                    build_fixed_part<L::C, L::R, L::S, BF16>(kpart, xs, cstride, rstride, a_hi, a_lo, swap);
                }
            }
            for (int kc = kpart; kc < nchunks && FX == 0 && !(p.debug & 16); kc += KPARTS) {
                const uint32_t ko = ptx::smem_u32(koff + kc * 32);
                uint32_t hv[16], lv[16];
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const int4 o = lds_v4(ko + 16 * q);
                    const float v0 = lds_f32(xs + o.x), v1 = lds_f32(xs + o.y);
                    const float v2 = lds_f32(xs + o.z), v3 = lds_f32(xs + o.w);
                    const uint32_t h01 = bf16x2_rn(v0, v1), h23 = bf16x2_rn(v2, v3);
                    hv[2 * q] = h01;
                    hv[2 * q + 1] = h23;
                    lv[2 * q] = bf16x2_rn(v0 - __uint_as_float(h01 << 16),
                                          v1 - __uint_as_float(h01 & 0xffff0000u));
                    lv[2 * q + 1] = bf16x2_rn(v2 - __uint_as_float(h23 << 16),
                                              v3 - __uint_as_float(h23 & 0xffff0000u));
                }
                if (!(p.debug & 2)) {
                    ptx::tmem_st_32x32b_x16(a_hi + kc * 16, hv);
                    ptx::tmem_st_32x32b_x16(a_lo + kc * 16, lv);
                }
            }
            if (lane == 0 && (warp == 0 || warp == 8)) ts_stamp(p, warp == 0 ? 3 : 13, i);
            // the next tile: origin and barrier tests, in flight over this tile's drain
            const int ws_cur = ws;
            tw.next(p);
            ++i;
            if (++ws == p.nwin) {
                ws = 0;
                wph ^= 1;
            }
            have = tw.t < p.total_tiles;
            const int bn = p.nab == 2 ? (i & 1) : 0;  // the next tile's A buffer and its use count
            const uint32_t aph = ((p.nab == 2 ? i >> 1 : i) & 1) ^ 1;
            bool s_ok = true, a_ok = true;
            if (have) {
                xs = window_origin(tw, ws);
                s_ok = ptx::mbar_test(&s_full[ws], wph);
                a_ok = ptx::mbar_test(&a_empty[bn], aph);
            }
            ptx::tmem_st_wait();
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0 && (warp == 0 || warp == 8)) ts_stamp(p, warp == 0 ? 4 : 14, i - 1);
            if (lane == 0) {
                if (CG == 2)
                    ptx::mbar_arrive_remote(a_full_l0 + b * sizeof(uint64_t));
                else
                    ptx::mbar_arrive(&a_full[b]);
                ptx::mbar_arrive(&s_empty[ws_cur]);
            }
            if (have) {
                if (!s_ok) ptx::mbar_wait(&s_full[ws], wph);
                if (lane == 0 && (warp == 0 || warp == 8)) ts_stamp(p, warp == 0 ? 1 : 11, i);
                if (!a_ok) ptx::mbar_wait(&a_empty[bn], aph);
                ptx::tc_fence_after();
            }
        }
    } else if (warp < TS_TMA_WARP) {
        // ============================ epilogue ==========================================
        // TMEM -> registers (+bias).  With tma_store: each 32-channel chunk goes to a
        // double-buffered [32][128] smem tile and one elected thread TMA-stores it (the TMA
        // unit keeps the HBM writes in flight); otherwise coalesced 128-byte stores.
        const int quad = warp & 3;
        const int m = quad * 32 + lane;
        const bool issuer = threadIdx.x == TS_EPI_WARP0 * 32;
        int i = 0, chunk = 0;
        for (TileWalk tw(p, unit0, nunits); tw.t < p.total_tiles; tw.next(p), ++i) {
            const int b = i & 1;
            const uint32_t ph = (i >> 1) & 1;
            const int n = tw.n;
            const int p0 = tw.ti * (TS_BM * CG) + (int)rank * TS_BM;
            const int pix = p0 + m;
            const bool valid = pix < g.PQ;
            float* dst = p.out + (int64_t)n * g.K * g.PQ + pix;
            ptx::mbar_wait(&acc_full[b], ph);
            ptx::tc_fence_after();
            if (threadIdx.x == TS_EPI_WARP0 * 32) ts_stamp(p, 7, i);
#pragma unroll 1
            for (int c0 = 0; c0 < g.K; c0 += 32, ++chunk) {
                uint32_t r[32];
                ptx::tmem_ld_32x32b_x32(tmem_base + ((uint32_t)(quad * 32) << 16) + b * p.n_pad + c0,
                                        r);
                ptx::tmem_ld_wait();
                if (c0 + 32 >= g.K) {  // accumulator fully in registers: release it early
                    ptx::tc_fence_before();
                    __syncwarp();
                    if (lane == 0) {  // (128 remote arrivals a tile serialise at the leader's barrier)
                        if (CG == 2)
                            ptx::mbar_arrive_remote(acc_empty_l0 + b * sizeof(uint64_t));
                        else
                            ptx::mbar_arrive(&acc_empty[b]);
                    }
                    if (threadIdx.x == TS_EPI_WARP0 * 32) ts_stamp(p, 8, i);
                }
                if (p.debug & 8) continue;
                if (p.tma_store) {
                    float* buf = ostage + (chunk & 1) * (32 * TS_BM);
                    if (issuer) ptx::bulk_wait_read<1>();  // the store 2 chunks ago left buf
                    asm volatile("bar.sync 1, 128;" ::: "memory");
                    const uint32_t bs = ptx::smem_u32(buf + m);
                    if (p.bias) {
#pragma unroll
                        for (int e = 0; e < 32; ++e)
                            sts_f32(bs + 4 * e * TS_BM, __uint_as_float(r[e]) +
                                                            (c0 + e < g.K ? __ldg(p.bias + c0 + e) : 0.f));
                    } else {
#pragma unroll
                        for (int e = 0; e < 32; ++e) sts_f32(bs + 4 * e * TS_BM, __uint_as_float(r[e]));
                    }
                    ptx::fence_proxy_async_smem();
                    asm volatile("bar.sync 1, 128;" ::: "memory");
                    if (issuer && p0 < g.PQ) {
                        ptx::tma_store_3d(&tm_y, buf, p0, c0, n);
                        ptx::bulk_commit();
                        ts_stamp(p, 9, i);
                    }
                } else if (valid) {
#pragma unroll
                    for (int e = 0; e < 32; ++e) {
                        const int co = c0 + e;
                        if (co < g.K)
                            dst[(int64_t)co * g.PQ] =
                                __uint_as_float(r[e]) + (p.bias ? __ldg(p.bias + co) : 0.f);
                    }
                }
            }
        }
        // the staging buffers must outlive the stores' reads; the kernel boundary completes the writes
        if (issuer) ptx::bulk_wait_read<0>();
    } else if (warp == TS_TMA_WARP) {
        // ============================ TMA: weights once, then input windows =============
        const uint32_t leader = ptx::elect_one();
        constexpr int WBLK = BF16 ? 64 : 32;  // reduction elements per 128-byte weight row block
        const int wblocks = p.kb_w / WBLK;
        // the weights are issued after the first window: the window heads the first tile's
        // chain (build -> MMA), the weights are first needed at the MMAs
        auto load_weights = [&]() {
            if (leader) {  // this CTA's weight rows [rank * w_rows, +w_rows); pairs: leader barrier
                if (rank == 0) ptx::mbar_arrive_expect_tx(w_full, CG * 2 * p.w_half_bytes);
                const int row0 = (int)rank * p.w_rows;
                for (int kb = 0; kb < wblocks; ++kb) {
                    uint8_t* dh = w_hi + (size_t)kb * p.w_rows * 128;
                    uint8_t* dl = w_lo + (size_t)kb * p.w_rows * 128;
                    if (CG == 2) {
                        ptx::tma_load_2d_pair(dh, &tm_whi, ptx::leader_bar(w_full), kb * WBLK, row0);
                        ptx::tma_load_2d_pair(dl, &tm_wlo, ptx::leader_bar(w_full), kb * WBLK, row0);
                    } else {
                        ptx::tma_load_2d(dh, &tm_whi, w_full, kb * WBLK, row0);
                        ptx::tma_load_2d(dl, &tm_wlo, w_full, kb * WBLK, row0);
                    }
                }
            }
        };
        __syncwarp();
        int i = 0;
        int ws = 0;  // staging-window ring slot and phase
        uint32_t wph = 0;
        for (TileWalk tw(p, unit0, nunits); tw.t < p.total_tiles; tw.next(p), ++i) {
            const int n = tw.n;
            const int p0 = min(tw.ti * (TS_BM * CG) + (int)rank * TS_BM, g.PQ - 1);
            const int iy0 = div_q(p0, p) * g.sh - g.ph;
            ptx::mbar_wait(&s_empty[ws], wph ^ 1);
            if (leader) ts_stamp(p, 0, i);
            if (leader && (p.debug & 4)) {
                ptx::mbar_arrive(&s_full[ws]);
            } else if (leader) {
                ptx::mbar_arrive_expect_tx(&s_full[ws], p.stage_bytes);
                ptx::tma_load_4d(reinterpret_cast<uint8_t*>(stage0) + (size_t)ws * p.stage_stride, &tm_x,
                                 &s_full[ws], -p.x0, iy0, 0, n);
            }
            if (i == 0) load_weights();
            __syncwarp();
            if (++ws == p.nwin) {
                ws = 0;
                wph ^= 1;
            }
        }
        if (i == 0) load_weights();  // a CTA without tiles (not launched by launch_conv_ts)
    } else {
        // ============================ MMA issuer ========================================
        const uint32_t leader = ptx::elect_one();
        const uint32_t idesc = ptx::idesc_f32acc<BF16>(TS_BM * CG, p.n_pad);
        const uint64_t dbh0 = ptx::sdesc_k_sw128(ptx::smem_u32(w_hi));
        const uint64_t dbl0 = ptx::sdesc_k_sw128(ptx::smem_u32(w_lo));
        const uint32_t blk16 = (uint32_t)(p.w_rows * 128) >> 4;  // one 64-wide K block of B
        const int ksteps = p.kp / (BF16 ? 16 : 8);  // one MMA covers 32 bytes of reduction per row
        if (rank == 0) ptx::mbar_wait(w_full, 0);
        int i = 0;
        for (TileWalk tw(p, unit0, nunits); tw.t < p.total_tiles && rank == 0; tw.next(p), ++i) {
            const int b = i & 1;  // accumulator
            const uint32_t ph = (i >> 1) & 1;
            if (!BF16 && p.khalves == 2) {  // two K halves per tile through the two A buffers
                ptx::mbar_wait(&acc_empty[b], ph ^ 1);
                const uint32_t d = tmem_base + b * p.n_pad;
                for (int h = 0; h < 2; ++h) {
                    ptx::mbar_wait(&a_full[h], (uint32_t)(i & 1));
                    ptx::tc_fence_after();
                    if (leader) ts_stamp(p, h ? 6 : 5, i);
                    const uint32_t a_hi = tmem_base + col_a0 + h * p.kp, a_lo = a_hi + p.kp / 2;
                    if (leader) {
                        for (int jj = 0; jj < ksteps / 2 && !(p.debug & 1); ++jj) {
                            const int j = h * (ksteps / 2) + jj;
                            if (j >= p.ksteps_real) break;  // all-zero padding steps
                            const uint64_t boff = (uint64_t)((j >> 2) * blk16 + (j & 3) * 2);
                            ptx::umma_ts<BF16>(d, a_lo + jj * 8, dbh0 + boff, idesc, j > 0 ? 1u : 0u);
                            ptx::umma_ts<BF16>(d, a_hi + jj * 8, dbl0 + boff, idesc, 1u);
                            ptx::umma_ts<BF16>(d, a_hi + jj * 8, dbh0 + boff, idesc, 1u);
                        }
                        ptx::umma_commit(&a_empty[h]);
                        if (h == 1) {
                            ptx::umma_commit(&acc_full[b]);
                            ts_stamp(p, 10, i);
                        }
                    }
                    __syncwarp();
                }
                continue;
            }
            const int ba = p.nab == 2 ? b : 0;  // A buffer and the parity of its use count
            const uint32_t pha = p.nab == 2 ? ph : (uint32_t)(i & 1);
            ptx::mbar_wait(&a_full[ba], pha);
            if (leader) ts_stamp(p, 5, i);
            ptx::mbar_wait(&acc_empty[b], ph ^ 1);
            ptx::tc_fence_after();
            if (leader) ts_stamp(p, 6, i);
            const uint32_t d = tmem_base + b * p.n_pad;
            const uint32_t a_hi = tmem_base + col_a0 + ba * p.acols;
            const uint32_t a_lo = a_hi + half_cols;
            if (leader) {
                for (int j = 0; j < min(ksteps, p.ksteps_real) && !(p.debug & 1); ++j) {
                    const uint64_t boff = (uint64_t)((j >> 2) * blk16 + (j & 3) * 2);
                    if (CG == 2) {
                        ptx::umma_ts_bf16_pair(d, a_lo + j * 8, dbh0 + boff, idesc, j > 0 ? 1u : 0u);
                        ptx::umma_ts_bf16_pair(d, a_hi + j * 8, dbl0 + boff, idesc, 1u);
                        ptx::umma_ts_bf16_pair(d, a_hi + j * 8, dbh0 + boff, idesc, 1u);
                    } else {
                        ptx::umma_ts<BF16>(d, a_lo + j * 8, dbh0 + boff, idesc, j > 0 ? 1u : 0u);
                        ptx::umma_ts<BF16>(d, a_hi + j * 8, dbl0 + boff, idesc, 1u);
                        ptx::umma_ts<BF16>(d, a_hi + j * 8, dbh0 + boff, idesc, 1u);
                    }
                }
                if (CG == 2) {
                    ptx::umma_commit_pair(&a_empty[ba]);
                    ptx::umma_commit_pair(&acc_full[b]);
                } else {
                    ptx::umma_commit(&a_empty[ba]);
                    ptx::umma_commit(&acc_full[b]);
                }
                ts_stamp(p, 10, i);
            }
            __syncwarp();
        }
    }

    ptx::tc_fence_before();
    if (CG == 2)
        ptx::cluster_sync();
    else
        __syncthreads();
    if (warp == TS_MMA_WARP) {
        ptx::tc_fence_after();
        if (CG == 2)
            ptx::tmem_dealloc_pair(tmem_base, TS_TMEM_COLS);
        else
            ptx::tmem_dealloc(tmem_base, TS_TMEM_COLS);
    }
}

// ----------------------------------------------------------------------------------------
// Host side
// ----------------------------------------------------------------------------------------
using TsKernel = void (*)(const TsParams, const CUtensorMap, const CUtensorMap, const CUtensorMap,
                         const CUtensorMap);
// the 3xTF32 kernels: compile-time layouts, single CTAs, plain or mixed reduction layout
static TsKernel ts_kernel_tf32(int fixed, int mode) {
    if (mode == 1) return nullptr;  // no padded-pair tf32 kernels (plan_ts never asks for one)
    switch (fixed) {
#define CB_TS_K(id, c, r, s)                                              \
    case id:                                                              \
        return mode == 3   ? conv_ts_kernel<1, id, 3, false>              \
               : mode == 2 ? conv_ts_kernel<1, id, 2, false>              \
                           : conv_ts_kernel<1, id, 0, false>;
        CB_TS_FIXED_LIST(CB_TS_K)
#undef CB_TS_K
        default: return nullptr;
    }
}

template <int CG>
static TsKernel ts_kernel_for(int fixed, int mode) {
    switch (fixed) {
#define CB_TS_K(id, c, r, s)                                       \
    case id:                                                       \
        return mode == 3   ? conv_ts_kernel<CG, id, 3>             \
               : mode == 2 ? conv_ts_kernel<CG, id, 2>             \
               : mode == 1 ? conv_ts_kernel<CG, id, 1>             \
                           : conv_ts_kernel<CG, id, 0>;
        CB_TS_FIXED_LIST(CB_TS_K)
#undef CB_TS_K
        default: return conv_ts_kernel<CG, 0, 0>;
    }
}

struct TsPlan {
    bool ok;
    int cg;  // 1: one CTA per 128-pixel tile; 2: CTA pairs (cta_group::2) on 256-pixel tiles
    int kp, n_pad, kb_w, box_rows, box_w, x0, pair, pf, kdim;
    uint32_t stage_bytes, stage_stride, w_half_bytes;
    int nwin;
    bool tma_store;
    size_t smem;
    bool bf16;
    int nab, acols;  // A buffers in TMEM and the columns of one
    int khalves;     // 2: the single tf32 buffer split into two half-K buffers
};

static int ts_fixed_id(const Geom& g) {
    if (g.dw != 1 || env("CB_TS_GENERIC")) return 0;
#define CB_TS_MATCH(id, c, r, s) \
    if (g.C == c && g.R == r && g.S == s) return id;
    CB_TS_FIXED_LIST(CB_TS_MATCH)
#undef CB_TS_MATCH
    return 0;
}

static TsPlan plan_ts(const Geom& g, bool bf16 = true) {
    TsPlan pl{};
    pl.bf16 = bf16;
    if (g.G != 1 || g.npix == 0) return pl;
    if (!bf16 && !ts_fixed_id(g)) return pl;  // the tf32 split: compile-time layouts only
    // int32 tile walk and the float pixel -> row division (TileWalk, div_q)
    if (g.PQ >= (1 << 21) || (int64_t)g.N * ((g.PQ + TS_BM - 1) / TS_BM) >= (1LL << 31) - 1024) return pl;
    pl.n_pad = round_up(g.K, 16);
    pl.x0 = round_up(g.pw, 4);  // 16-byte aligned window start
    // pair mode: compile-time producer, even horizontal stride, odd S, the padded reduction
    // fits TMEM next to two accumulators
    // (2: the mixed layout -- tap pairs plus one single tap per row, no padding; 1: padded
    // pairs, kept for A/B runs with CB_TS_PAIRMODE=1)
    pl.pair = 0;
    pl.pf = (pl.x0 - g.pw) & 1;
    const int pair_mode = [] {  // read per call: the tests switch layouts in-process
        const char* e = env("CB_TS_PAIRMODE");
        return env("CB_TS_NO_PAIR") ? 0 : e ? std::atoi(e) : 2;
    }();
    const int pm = (pair_mode == 1 && !bf16) ? 2 : pair_mode;  // no padded-pair tf32 kernels
    const int kd_pair = pm == 2 ? mixed_kdim(g.C * g.R, g.S) : g.C * g.R * (g.S + 1);
    // one A buffer holds hi and lo halves: kp / 2 + kp / 2 columns of bf16 pairs, kp + kp of tf32 words
    const int per_el = bf16 ? 1 : 2;
    if (pm && ts_fixed_id(g) && g.S % 2 == 1 && g.sw % 2 == 0 &&
        2 * pl.n_pad + (bf16 ? 2 : 1) * per_el * round_up(kd_pair, 32) <= TS_TMEM_COLS)
        pl.pair = pm == 2 ? 2 : 1;
    pl.kdim = pl.pair ? kd_pair : g.kdim;
    pl.kp = round_up(pl.kdim, 32);
    pl.kb_w = round_up(pl.kdim, 64);  // == cb_split_kdim(kdim)
    pl.acols = per_el * pl.kp;
    pl.nab = 2 * pl.n_pad + 2 * pl.acols <= TS_TMEM_COLS ? 2 : 1;  // tf32 words: often one buffer only
    if (pl.n_pad > 256 || 2 * pl.n_pad + pl.nab * pl.acols > TS_TMEM_COLS) return pl;
    pl.khalves = (!bf16 && pl.nab == 1 && CB_TS_KPARTS == 1 && !env("CB_TS_NO_HALVES")) ? 2 : 1;
    // window columns: every tap of every output column (+ the pad tap past the last one)
    const int need = (g.Q - 1) * g.sw + (pl.x0 - g.pw) + (g.S - 1) * g.dw + 1 + (pl.pair == 1 && !pl.pf ? 1 : 0);
    pl.box_w = round_up(std::max(g.W + g.pw + pl.x0, need), 4);
    const int out_rows = std::min(g.P, (TS_BM - 1) / std::max(1, g.Q) + 2);
    pl.box_rows = (out_rows - 1) * g.sh + (g.R - 1) * g.dh + 1;
    if (pl.box_w > 256 || pl.box_rows > 256 || g.C > 256 || (g.W % 4) != 0) return pl;
    pl.stage_bytes = (uint32_t)g.C * pl.box_rows * pl.box_w * 4;
    pl.stage_stride = (pl.stage_bytes + 1023) / 1024 * 1024;
    // CTA pairs halve each SM's weight reads (the B operand, ~30% of the shared-memory
    // traffic of a tile): N split N/2 per CTA, needs N/2 a multiple of 16 (SW128 atoms)
    pl.cg = 1;
    {
        const char* e = env("CB_TS_CG");
        const int want = e ? std::atoi(e) : 1;  // pairs measured slower on cfg3 (30 vs 22 us)
        if (want == 2 && bf16 && pl.n_pad % 32 == 0 && pl.n_pad <= 256) pl.cg = 2;
    }
    pl.w_half_bytes = (uint32_t)(pl.n_pad / pl.cg) * pl.kb_w * (bf16 ? 2 : 4);
    // >= 120 KB keeps one CTA per SM (each allocates all 512 TMEM columns)
    pl.tma_store = (g.PQ % 4) == 0;  // 16-byte global strides for the output map
    auto smem_for = [&](int nwin) {
        return std::max<size_t>(120 * 1024, 1024 + 2 * (size_t)pl.w_half_bytes +
                                                nwin * (size_t)pl.stage_stride + 1024 +
                                                2 * 32 * TS_BM * 4 + 4 * (size_t)pl.kp);
    };
    static const int max_win = [] {
        const char* e = std::getenv("CB_TS_NWIN");
        return e ? std::max(2, std::min(4, std::atoi(e))) : 4;
    }();
    pl.nwin = 2;
    while (pl.nwin < max_win && smem_for(pl.nwin + 1) <= 227 * 1024) ++pl.nwin;
    pl.smem = smem_for(pl.nwin);
    pl.ok = pl.stage_bytes <= 64 * 1024 && pl.smem <= 227 * 1024;
    return pl;
}

// Used by fused_layout: the direct kernel serves this descriptor (bf16 split only).
bool ts_eligible(const Geom& g, bool bf16) { return plan_ts(g, bf16).ok; }

// The K7 weight layout: reduction length of the packed rows (C*R*(S+1) in pair mode) and,
// in pair mode, the pad position (*pf = 1: pad tap first in each (c, r) row).
int ts_weight_kdim(const Geom& g, bool bf16, int* pair, int* pf) {
    const TsPlan pl = plan_ts(g, bf16);
    *pair = pl.pair;
    *pf = pl.pf;
    return pl.pair ? pl.kdim : g.kdim;
}

// The K7 reduction layout, element by element: map[k] = the OIHW index (c*R + r)*S + s of the
// weight / window tap at reduction position k, or -1 for a zero element (pad taps, the tail).
// Returns the layout's length (ts_weight_kdim), or -1 when K7 does not serve the descriptor.
int ts_reduction_map(const Geom& g, bool bf16, int cap, int32_t* map) {
    const TsPlan pl = plan_ts(g, bf16);
    if (!pl.ok) return -1;
    const int kd = pl.pair ? pl.kdim : g.kdim;
    for (int k = 0; k < kd && k < cap; ++k) {
        int v = -1;
        if (pl.pair == 2) {
            const MixedTap t = mixed_map(k, g.C * g.R, g.S, pl.pf);
            if (t.cr >= 0) v = t.cr * g.S + t.s;
        } else if (pl.pair == 1) {
            const int cr = k / (g.S + 1), s = k - cr * (g.S + 1) - pl.pf;
            if (s >= 0 && s < g.S) v = cr * g.S + s;
        } else {
            v = k;
        }
        map[k] = v;
    }
    return kd;
}

int ts_plan_query(const Geom& g, bool bf16, cb_tile_plan* out) {
    const TsPlan pl = plan_ts(g, bf16);
    if (!pl.ok) return fail(CB_ERR_UNSUPPORTED, "direct TMEM conv does not fit this descriptor");
    const int64_t tiles = (int64_t)g.N * ((g.PQ + TS_BM * pl.cg - 1) / (TS_BM * pl.cg));
    out->variant = bf16 ? CB_VARIANT_TC3XBF16 : CB_VARIANT_TC3XTF32;
    out->block_m = TS_BM * pl.cg;
    out->block_n = pl.n_pad;
    out->block_k = bf16 ? 16 : 8;
    out->stages = pl.nab;
    out->splits = 1;
    out->m_tiles = tiles;
    out->n_tiles = 1;
    out->k_blocks = pl.kp / (bf16 ? 16 : 8);
    out->ctas = (int)std::min<int64_t>(tiles, sm_count() / pl.cg) * pl.cg;
    return CB_OK;
}

static PFN_cuTensorMapEncodeTiled_v12000 ts_encode_fn() {
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

unsigned long long* debug_trace_buffer(int ctas, cudaStream_t st);

int launch_conv_ts(const Geom& g, bool bf16, const float* x, const void* w_hi, const void* w_lo,
                   const float* bias, float* y, cudaStream_t st) {
    const TsPlan pl = plan_ts(g, bf16);
    if (!pl.ok) return fail(CB_ERR_UNSUPPORTED, "direct TMEM conv does not fit this descriptor");
    auto enc = ts_encode_fn();
    if (!enc) return fail(CB_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    if ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(w_hi) |
         reinterpret_cast<uintptr_t>(w_lo)) & 15)
        return fail(CB_ERR_MISALIGNED, "input and packed weights must be 16-byte aligned");
    CUtensorMap mx, mwh, mwl, my{};
    {
        cuuint64_t dims[4] = {(cuuint64_t)g.W, (cuuint64_t)g.H, (cuuint64_t)g.C, (cuuint64_t)g.N};
        cuuint64_t strides[3] = {(cuuint64_t)g.W * 4, (cuuint64_t)g.HW * 4,
                                 (cuuint64_t)g.C * g.HW * 4};
        cuuint32_t box[4] = {(cuuint32_t)pl.box_w, (cuuint32_t)pl.box_rows, (cuuint32_t)g.C, 1};
        cuuint32_t es[4] = {1, 1, 1, 1};
        CUresult r = enc(&mx, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(x), dims,
                         strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS)
            return fail(CB_ERR_CUDA, "cuTensorMapEncodeTiled (input) failed: " + std::to_string((int)r));
    }
    for (int h = 0; h < 2; ++h) {
        cuuint64_t dims[2] = {(cuuint64_t)pl.kb_w, (cuuint64_t)g.K};
        cuuint64_t strides[1] = {(cuuint64_t)pl.kb_w * (bf16 ? 2 : 4)};
        cuuint32_t box[2] = {bf16 ? 64u : 32u, (cuuint32_t)(pl.n_pad / pl.cg)};  // 128-byte rows
        cuuint32_t es[2] = {1, 1};
        CUresult r = enc(h ? &mwl : &mwh, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                         const_cast<void*>(h ? w_lo : w_hi), dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS)
            return fail(CB_ERR_CUDA, "cuTensorMapEncodeTiled (weights) failed: " + std::to_string((int)r));
    }
    if (pl.tma_store) {
        if (reinterpret_cast<uintptr_t>(y) & 15)
            return fail(CB_ERR_MISALIGNED, "output must be 16-byte aligned");
        cuuint64_t dims[3] = {(cuuint64_t)g.PQ, (cuuint64_t)g.K, (cuuint64_t)g.N};
        cuuint64_t strides[2] = {(cuuint64_t)g.PQ * 4, (cuuint64_t)g.K * g.PQ * 4};
        cuuint32_t box[3] = {(cuuint32_t)TS_BM, 32, 1};
        cuuint32_t es[3] = {1, 1, 1};
        CUresult r = enc(&my, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, y, dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                         CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS)
            return fail(CB_ERR_CUDA, "cuTensorMapEncodeTiled (output) failed: " + std::to_string((int)r));
    }
    TsParams prm{};
    prm.tma_store = pl.tma_store ? 1 : 0;
    if (env("CB_TS_NO_TMA_STORE")) prm.tma_store = 0;
    prm.g = g;
    prm.bias = bias;
    prm.out = y;
    prm.kp = pl.kp;
    prm.n_pad = pl.n_pad;
    prm.kb_w = pl.kb_w;
    prm.tiles_per_img = (g.PQ + TS_BM * pl.cg - 1) / (TS_BM * pl.cg);
    prm.inv_q = 1.0f / (float)g.Q;
    prm.fixed = ts_fixed_id(g);
    prm.pair = pl.pair;
    prm.pf = pl.pf;
    prm.total_tiles = (int64_t)g.N * prm.tiles_per_img;
    prm.box_rows = pl.box_rows;
    prm.box_w = pl.box_w;
    prm.x0 = pl.x0;
    prm.stage_bytes = pl.stage_bytes;
    prm.stage_stride = pl.stage_stride;
    prm.nwin = pl.nwin;
    prm.nab = pl.nab;
    prm.acols = pl.acols;
    prm.khalves = pl.khalves;
    prm.ksteps_real = env("CB_TS_ALL_KSTEPS") ? pl.kp : (pl.kdim + (bf16 ? 15 : 7)) / (bf16 ? 16 : 8);
    prm.w_half_bytes = pl.w_half_bytes;
    prm.w_rows = pl.n_pad / pl.cg;
    if (const char* dbg = env("CB_TS_DEBUG")) prm.debug = std::atoi(dbg);
    if (env("CB_TS_TRACE")) prm.trace = debug_trace_buffer(1024, st);
    const int mode = pl.pair == 2 ? 2 + pl.pf : pl.pair;
    const TsKernel kern = !bf16 ? ts_kernel_tf32(prm.fixed, mode)
                          : pl.cg == 2 ? ts_kernel_for<2>(prm.fixed, mode) : ts_kernel_for<1>(prm.fixed, mode);
    if (!kern) return fail(CB_ERR_UNSUPPORTED, "direct TMEM conv: no tf32 kernel for this layout");
    {
        static std::mutex mu;
        static std::set<const void*> ready;  // kernels whose smem attribute is set
        std::lock_guard<std::mutex> lk(mu);
        if (!ready.count(reinterpret_cast<const void*>(kern))) {
            const cudaError_t attr_err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
            if (attr_err != cudaSuccess)
                return fail(CB_ERR_CUDA, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(attr_err));
            ready.insert(reinterpret_cast<const void*>(kern));
        }
    }
    const int units = (int)std::min<int64_t>(prm.total_tiles, sm_count() / pl.cg);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)(units * pl.cg));
    cfg.blockDim = dim3(TS_THREADS);
    cfg.dynamicSmemBytes = pl.smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    int nattr = 0;
    static const bool pdl = std::getenv("CB_NO_PDL") == nullptr;
    if (pdl) {  // the prologue may overlap the stream predecessor (grid_dependency_wait)
        attr[nattr].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[nattr].val.programmaticStreamSerializationAllowed = 1;
        ++nattr;
    }
    if (pl.cg == 2) {  // no cluster attribute for single CTAs
        attr[nattr].id = cudaLaunchAttributeClusterDimension;
        attr[nattr].val.clusterDim.x = pl.cg;
        attr[nattr].val.clusterDim.y = 1;
        attr[nattr].val.clusterDim.z = 1;
        ++nattr;
    }
    cfg.attrs = attr;
    cfg.numAttrs = nattr;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, prm, mx, mwh, mwl, my);
    if (e != cudaSuccess) return fail(CB_ERR_CUDA, std::string("conv_ts launch: ") + cudaGetErrorString(e));
    return check_launch("conv_ts_kernel");
}

}  // namespace cb
