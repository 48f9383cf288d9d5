// cb_common.cuh -- shared host/device helpers for libconvb200 (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <string>

#include "convb200.h"

namespace cb {

// Environment switches on launch paths (CB_*): looked up in a per-thread snapshot of the
// process environment's CB_ entries, taken once per C-ABI call (make_geom and the entry
// points without a descriptor refresh it), instead of one libc getenv per switch -- a K6
// launch reads ~17 switches and every getenv walks the whole environment (~0.3 us each in a
// typical process, half of the call's host time).  Same result as getenv at the time of the
// refresh, so in-process toggles (the tests) take effect at the next call.
void env_refresh();
const char* env(const char* name);


// Diagnostics timelines (CB_TMA_TRACE / CB_TS_TRACE / CB_K8_TRACE) exist only in a build with
// -DCB_TRACE (build(defines=("-DCB_TRACE",)), loaded with CB_LIB_PATH): in the product build
// every stamp and the conditions around it compile away.
#ifdef CB_TRACE
constexpr bool kTrace = true;
#else
constexpr bool kTrace = false;
#endif

// ------------------------------------------------------------------------------------
// Error reporting (thread-local; returned through cb_last_error_string()).
// ------------------------------------------------------------------------------------
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int check_launch(const char* what);

// ------------------------------------------------------------------------------------
// Conv geometry, resolved once on the host and passed by value to kernels.
// Mirrors output_shape (descriptor.py:84-92): floor semantics.
// ------------------------------------------------------------------------------------
struct Geom {
    int N, C, H, W, K, R, S;
    int sh, sw, ph, pw, dh, dw, G;
    int P, Q;        // output spatial dims
    int cpg, kpg;    // channels / output channels per group
    int kdim;        // cpg * R * S  (GEMM reduction length per group)
    int kdim_pad;    // cb_split_kdim(kdim)
    int PQ, HW, RS;
    int64_t npix;    // N * P * Q
};

int make_geom(const cb_conv_desc* d, Geom* g);  // CB_OK or CB_ERR_INVALID

inline int32_t round_up(int32_t a, int32_t b) { return (a + b - 1) / b * b; }
inline int64_t ceil_div64(int64_t a, int64_t b) { return (a + b - 1) / b; }

int sm_count();  // cached multiProcessorCount of the current device
// Reduction elements accumulated in one tensor-core accumulator before it is drained and
// added in fp32 (round to nearest) by the epilogue: the tcgen05 fp32 accumulation truncates,
// so its error grows faster than linearly with the MMAs per accumulator.  CB_PROMOTE_K
// overrides (diagnostics; 0 = never promote).
int promote_k(bool bf16);  // defaults: 2048 (tf32 MMAs, K = 8 each), 4096 (bf16 MMAs, K = 16)

// ------------------------------------------------------------------------------------
// Pixel addressing modes shared by the GEMM/conv kernels.
//
// Every kernel walks "pixels" j in [0, npix) (the GEMM column / TMEM lane dimension)
// and "reduction" k in [0, kdim).  Source (activation-side) operands are either
// gathered from NCHW (implicit im2col) or linear in k per pixel:
//     addr(j, k) = base(j) + k * kstride(j)
// which covers the im2col matrix (base=j, kstride=ld).  The SConv slice buffer of a
// chunk is such a matrix too: the im2col columns of the chunk's pixels [jb, jb+J),
// (k, pixel) with row stride J, so the SConv GEMM runs in matrix mode with launch-local
// pixels.  Outputs are always linear:
//     out(j, f) = obase(j) + f * okstride(j)
// covering NCHW (obase = n*K*PQ + p, okstride = PQ) and a row-major matrix (the SConv
// accumulators of a chunk: (f, pixel), row stride J).
// ------------------------------------------------------------------------------------
enum SrcMode : int { SRC_CONV = 0, SRC_MATRIX = 1 };
enum DstMode : int { DST_NCHW = 0, DST_MATRIX = 1 };

struct PixMap {
    int src_mode, dst_mode;
    int64_t src_ld;      // SRC_MATRIX row stride (group g starts at row g*kdim)
    int64_t dst_ld;      // DST_MATRIX row stride
    int64_t j_begin;     // first pixel of this launch
    int64_t j_count;     // pixels processed by this launch
};

// Linear source address components for pixel j (SRC_MATRIX).
__device__ __forceinline__ void src_linear(const Geom& g, const PixMap& pm, int64_t j,
                                           int64_t& base, int64_t& kstride) {
    base = j;
    kstride = pm.src_ld;
}

// Output address components for pixel j.
__device__ __forceinline__ void dst_linear(const Geom& g, const PixMap& pm, int64_t j,
                                           int64_t& base, int64_t& okstride) {
    if (pm.dst_mode == DST_NCHW) {
        int64_t n = j / g.PQ;
        int64_t p = j - n * g.PQ;
        base = n * (int64_t)g.K * g.PQ + p;
        okstride = g.PQ;
    } else {
        base = j;
        okstride = pm.dst_ld;
    }
}

// ------------------------------------------------------------------------------------
// Reduction layout of the TMA-fed fused conv (conv_tma.cu).  The reduction runs over
// (tap r*S+s, channel chunk cb, channel ci) with CB channels per chunk; one pipeline stage
// is 128 bytes of reduction per pixel row = cps chunks.  Activations live in an NHWC
// split workspace with a c_alloc channel pitch (16-byte aligned pixels).
// ------------------------------------------------------------------------------------
struct FusedLayout {
    int tma;           // 1: TMA im2col path usable, 0: use the gather kernel
    int eb;            // operand bytes: 4 (tf32) / 2 (bf16)
    int c_alloc;       // NHWC channel pitch (elements)
    int cb;            // channels per chunk (power of two)
    int chunk_bytes;   // cb * eb: 16, 32, 64 or 128
    int chk;           // chunks per tap
    int cps;           // chunks per stage (128 / chunk_bytes)
    int total_chunks;  // R * S * chk
    int num_kb;        // pipeline stages (k blocks) per tile
    int kw_pad;        // weight row length (elements) = num_kb * 128 / eb
    int64_t act_elems; // N * H * W * c_alloc (per hi / lo buffer)
    int fold;          // 0, or the kernel width S when the horizontal taps are folded into
                       // the channels (small C): the kernel then runs fold_geom(g)
    int ts;            // 1: the direct TMEM kernel (K7, conv_ts.cu) serves it (tma = 0)
    int stack;         // stacked taps (K9 sums the shifted planes): 0 none, 1 all R*S taps
                       // (kernel: stack_geom(g, 1)), 2 the S horizontal taps (stack_geom(g, 2))
};

// Tap stacking (few output channels, many input channels).  mode 1: all R*S taps become
// output channels of a 1x1 conv over the input grid, Y'[n][rs*K + f][h][w] = sum_c
// x[n][c][h][w] * w[f][c][r][s], and y[n][f][oy][ox] = sum_rs Y'[n][rs*K + f][oy*sh - ph +
// r*dh][ox*sw - pw + s*dw].  mode 2: only the S horizontal taps are stacked -- an R x 1 conv
// (vertical stride / pad / dilation kept) over all input columns, Y'[n][s*K + f][oy][w], and
// y[n][f][oy][ox] = sum_s Y'[n][s*K + f][oy][ox*sw - pw + s*dw].  x is read once per
// remaining tap instead of once per tap, and the MMA N grows by the stacked tap count.
// groups == 1 only.
inline Geom stack_geom(const Geom& g, int mode) {
    Geom t = g;
    if (mode == 1) {
        t.K = g.R * g.S * g.K;
        t.R = 1;
        t.sh = 1;
        t.ph = 0;
        t.dh = 1;
        t.P = g.H;
    } else {
        t.K = g.S * g.K;
    }
    t.kpg = t.K;
    t.S = 1;
    t.sw = 1;
    t.pw = 0;
    t.dw = 1;
    t.Q = g.W;
    t.PQ = t.P * t.Q;
    t.RS = t.R;
    t.kdim = g.cpg * t.R;
    t.kdim_pad = (t.kdim + 63) / 64 * 64;
    t.npix = (int64_t)g.N * t.PQ;
    return t;
}

// The same convolution with its S horizontal taps folded into the channel axis: the input
// becomes [N][H][Q][S*C] (x at column ox*sw + s*dw - pw for channel s*C + c, zero outside)
// and the kernel an R x 1 conv with unit horizontal stride and no horizontal padding.  Only
// for groups == 1.  P, Q, K, the reduction length and the output are unchanged.
inline Geom fold_geom(const Geom& g) {
    Geom f = g;
    f.C = g.C * g.S;
    f.cpg = f.C;
    f.W = g.Q;
    f.S = 1;
    f.sw = 1;
    f.pw = 0;
    f.dw = 1;
    f.HW = f.H * f.W;
    f.RS = f.R;
    f.kdim = f.cpg * f.R;
    return f;
}

// first pixel of slice s (slices of one image are consecutive bands of band_rows rows)
inline int64_t slice_pixel_begin(const Geom& g, int band_rows, int64_t s) {
    const int64_t per_img = (g.P + band_rows - 1) / band_rows;
    const int64_t n = s / per_img, b = s - n * per_img;
    if (n >= g.N) return g.npix;
    return n * g.PQ + b * band_rows * (int64_t)g.Q;
}

// ------------------------------------------------------------------------------------
// Precision splits.  tf32: 1 sign, 8 exponent, 10 mantissa bits, stored in an fp32
// container with the low 13 bits zero.  cvt.rna = round to nearest, ties away.
// ------------------------------------------------------------------------------------
__device__ __forceinline__ float tf32_rna(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

struct Split2 {
    float hi, lo;
};
__device__ __forceinline__ Split2 split_tf32(float x) {
    float hi = tf32_rna(x);
    float lo = tf32_rna(x - hi);
    return {hi, lo};
}

// bf16 round-to-nearest-even of an fp32 value, returned as raw bits.
__device__ __forceinline__ uint16_t bf16_rn_bits(float x) {
    uint16_t r;
    asm("cvt.rn.bf16.f32 %0, %1;" : "=h"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float bf16_bits_to_f32(uint16_t b) {
    return __uint_as_float(((uint32_t)b) << 16);
}

// ------------------------------------------------------------------------------------
// K7 "mixed" reduction layout (odd S = 2h + 1, even horizontal stride): every (c, r) row
// cr contributes h tap pairs -- (pf, pf + 1), (pf + 2, pf + 3), ... -- each one 8-byte
// aligned LDS.64 of two adjacent window columns, and one single tap (s = S - 1 when
// pf = 0, s = 0 when pf = 1).  Rows are laid out two at a time: the pairs of row 2j, the
// pairs of row 2j + 1, then the two singles as one more k pair, 2S elements per row pair
// with no padding; an odd last row is followed by one zero element.  Shared by the A
// producer (conv_ts.cu) and the weight packer (pack_kernels.cu).
//   mixed_kdim = NR * S + (NR & 1);  mixed_map(k) -> row cr and tap s, or cr = -1 (zero)
// ------------------------------------------------------------------------------------
struct MixedTap {
    int cr, s;
};
__host__ __device__ constexpr int mixed_kdim(int nr, int S) { return nr * S + (nr & 1); }
__host__ __device__ constexpr MixedTap mixed_map(int k, int nr, int S, int pf) {
    const int h2 = S - 1;  // pair elements of one row
    const int rp = k / (2 * S), o = k - rp * 2 * S;
    const int single = pf ? 0 : S - 1;
    if (2 * rp + 1 < nr) {
        if (o < h2) return {2 * rp, o + pf};
        if (o < 2 * h2) return {2 * rp + 1, o - h2 + pf};
        return {2 * rp + (o - 2 * h2), single};
    }
    if (2 * rp >= nr) return {-1, 0};
    if (o < h2) return {nr - 1, o + pf};
    if (o == h2) return {nr - 1, single};
    return {-1, 0};
}

}  // namespace cb
