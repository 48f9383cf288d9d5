/*
 * convb200.h -- C ABI of libconvb200.so, the B200 (sm_100a) 2D-convolution hot path.
 *
 * This is the drop-in boundary for the ConvBench (arXiv 2407.10730) algorithms.
 * The reference is pure Python/NumPy, so it has no FFI of its own; every entry
 * point below replaces one reference function (cited file:line, relative to
 * /root/reference/pkg/src/convbench/) and is bound from Python with ctypes by
 * paper_2407_10730_b200/_capi.py (see INTEGRATION.md for the binding).
 *
 * Conventions
 *   - Plain pointers and sizes only. Every float pointer is DEVICE memory owned by
 *     the caller; the library never allocates and never frees.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *     Calls are stream-ordered and asynchronous: no host synchronisation inside.
 *   - Layouts: activations NCHW fp32, weights OIHW fp32 (K, C/groups, R, S),
 *     bias (K,) or NULL, output NCHW fp32.  "cols" is the im2col matrix of
 *     im2col_transform (algos.py:99-121): row (c,ky,kx), column (n,oy,ox).
 *   - Every function returns a cb_status; on failure cb_last_error_string()
 *     (thread-local) says why.  The Python shim maps codes onto the reference
 *     exception types (InvalidDescriptorError, UnsupportedDescriptorError,
 *     ValueError, MemoryError, RuntimeError).
 */
#ifndef CONVB200_H
#define CONVB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CB_ABI_VERSION 1

typedef enum cb_status {
    CB_OK = 0,
    CB_ERR_INVALID = 1,      /* descriptor cannot describe a conv   (descriptor.py:23-24, :45-59) */
    CB_ERR_UNSUPPORTED = 2,  /* algorithm cannot run this descriptor (algos.py:35-36, :277-280)   */
    CB_ERR_WORKSPACE = 3,    /* a caller buffer is too small                                      */
    CB_ERR_MISALIGNED = 4,   /* pointer not 16-byte aligned where the kernel needs it             */
    CB_ERR_CUDA = 5          /* CUDA launch/runtime error (see cb_last_error_string)              */
} cb_status;

/* POD mirror of ConvDescriptor (descriptor.py:27-43); has_bias is 0/1. */
typedef struct cb_conv_desc {
    int32_t batch, in_channels, in_h, in_w, out_channels, k_h, k_w;
    int32_t stride_h, stride_w, pad_h, pad_w, dil_h, dil_w, groups, has_bias;
} cb_conv_desc;

/* SConv slice plan: a slice is one band of `band_rows` output rows over the full
 * output width of one image (the GPU counterpart of _TilePlan, algos.py:247-262).
 * Slices tile the (n, oy, ox) pixel range contiguously.  The SConv calls take a slice
 * range [first_slice, first_slice + count) = pixels [jb, je), J = je - jb.  Its slice
 * buffer is the (C*R*S) x J matrix of the range's im2col columns, laid out (k, pixel) with
 * row stride J: the slice holding pixels [j0, j0+np) is the column block [j0-jb, j0-jb+np)
 * (panels of consecutive slices are adjacent, so the GEMM's 128-pixel tiles run across
 * slice boundaries).  The accumulators are likewise a K x J matrix, (f, pixel).  Ranges are
 * processed as chunks sized for the grid. */
typedef struct cb_slice_plan {
    int32_t band_rows;   /* output rows per slice (last band of an image may be shorter) */
    int32_t num_slices;  /* batch * ceil(out_h / band_rows)                              */
} cb_slice_plan;

/* Tile decomposition the GEMM/conv kernels will use for a launch (IN_TILING). */
typedef struct cb_tile_plan {
    int32_t variant;     /* cb_variant                                                   */
    int32_t block_m;     /* pixels per CTA tile (TMEM lanes)                             */
    int32_t block_n;     /* output channels per CTA tile (TMEM fp32 columns)             */
    int32_t block_k;     /* reduction elements per pipeline stage                        */
    int32_t stages;      /* shared-memory pipeline depth                                 */
    int32_t splits;      /* split-K factor (grid.z)                                      */
    int64_t m_tiles, n_tiles, k_blocks, ctas;
} cb_tile_plan;

/* Compute-variant selector for the GEMM / fused entry points. */
typedef enum cb_variant {
    CB_VARIANT_TC3XTF32 = 0, /* tcgen05 kind::tf32, 3 products (hi*hi + hi*lo + lo*hi)   */
    CB_VARIANT_FFMA = 1,     /* SIMT fp32 FFMA                                           */
    CB_VARIANT_TC3XBF16 = 2  /* tcgen05 kind::f16 (bf16), 3 products; fp32-grade error    */
} cb_variant;

/* ---- library info ------------------------------------------------------------------ */
int         cb_version(void);
const char* cb_last_error_string(void);
int         cb_device_sm_count(int* sm_count);
/* Total kernels this library has launched in the process (for launch accounting). */
uint64_t    cb_launch_count(void);

/* ---- phase timing (replaces PhaseLedger's host clock, timing.py:28-151) -------------
 * Timing-enabled CUDA events as opaque handles, recorded on the caller's stream.  The
 * device-timed ledger brackets each phase with a pair; elapsed_ns waits for `end`.
 * `external` = 1 records inside a CUDA-graph capture (the graph re-records on replay). */
int cb_event_create(void** event);
int cb_event_destroy(void* event);
int cb_event_record(void* event, void* stream, int external);
int cb_event_elapsed_ns(void* start, void* end, int64_t* ns);

/* Hash of the CB_* diagnostics switches in the process environment (their names and
 * values): the key host-side callers put on cached layouts and plans, since the switches
 * change both.  One pass over environ. */
uint64_t cb_env_fingerprint(void);

/* output_shape (descriptor.py:84-92) with the same validation as ConvDescriptor. */
int cb_output_shape(const cb_conv_desc* d, int32_t* out_h, int32_t* out_w);

/* Bytes of caller scratch an algorithm needs (0 = none).
 *   algo 0: im2col-GEMM (cols matrix)
 *   algo 1: SConv slices + slice accumulators for ALL slices (a chunked run needs
 *           only (C*R*S + K) * 4 bytes per pixel of its largest chunk)
 *   algo 2: fused implicit GEMM (none) */
int cb_workspace_bytes(const cb_conv_desc* d, int algo, const cb_slice_plan* plan, size_t* bytes);

/* ---- K1: im2col packing, bit-exact copy. Replaces im2col_transform (algos.py:99-121).
 * cols must hold (C*R*S) x (N*P*Q) floats. */
int cb_im2col_f32(const cb_conv_desc* d, const float* x, float* cols, void* stream);

/* ---- SConv plan + K2 slice packing. Replaces _plan_tiles (algos.py:254-262) and the
 * per-tile pack loop (algos.py:305-324).  Slice data is bit-identical to the matching
 * im2col columns.  max_slice_pixels bounds band_rows * out_w (>= out_w is honoured).
 * cb_sconv_range returns the pixel range [*pix_begin, *pix_begin + *pix_count) of a
 * slice range. */
int cb_sconv_plan(const cb_conv_desc* d, int32_t max_slice_pixels, cb_slice_plan* plan);
int cb_sconv_range(const cb_conv_desc* d, const cb_slice_plan* plan, int32_t first_slice,
                   int32_t count, int64_t* pix_begin, int64_t* pix_count);
int cb_sconv_pack_f32(const cb_conv_desc* d, const cb_slice_plan* plan, int32_t first_slice,
                      int32_t count, const float* x, float* slices, void* stream);

/* ---- IN_TILING: the tile plan cb_conv_gemm_cols / cb_sconv_gemm use for
 * `pixels` output pixels (<= 0: the whole batch).  Pure host computation. */
int cb_plan_tiles(int variant, const cb_conv_desc* d, int64_t pixels, cb_tile_plan* plan);

/* ---- K3: weight split / reorder. Replaces the wmat reshape (algos.py:202, :291) and
 * _pack_a_panels (algos.py:124-130).  w is rows x kdim row-major; hi/lo are
 * rows x kdim_pad (kdim_pad = cb_split_kdim(kdim)), zero padded, with
 * hi = tf32_rn(w), lo = tf32_rn(w - hi).  For CB_VARIANT_TC3XBF16 the halves are bf16
 * (hi = bf16_rn(w), lo = bf16_rn(w - hi)) packed as uint16 in the same row layout;
 * pass the float pointers reinterpreted. */
int32_t cb_split_kdim(int32_t kdim);
int cb_weight_split(int variant, int32_t rows, int32_t kdim, const float* w, void* w_hi,
                    void* w_lo, void* stream);

/* ---- K4: GEMM on packed operands.  Replaces gemm (algos.py:142-182):
 *   c[i, j] (+)= sum_k a[i, k] * b[k, j]     a: m x k (pre-split by cb_weight_split
 *   for the TC variants, raw fp32 row-major for FFMA), b: k x n with row stride ldb,
 *   c: m x n with row stride ldc.  accumulate=1 adds to c's contents (the caller's
 *   initialisation, algos.py:158); accumulate=0 overwrites. */
int cb_gemm(int variant, int32_t m, int32_t n, int32_t k, const void* a_hi, const void* a_lo,
            const float* a_f32, const float* b, int64_t ldb, float* c, int64_t ldc,
            int accumulate, void* stream);

/* ---- K4 for the im2col path: y = conv via cols (K1 output) x weights, NCHW epilogue
 * with bias.  The GEMM + write-back of conv_baseline_im2col_gemm (algos.py:200-208). */
int cb_conv_gemm_cols(int variant, const cb_conv_desc* d, const float* cols, const void* w_hi,
                      const void* w_lo, const float* w_f32, const float* bias, float* y,
                      void* stream);

/* ---- K4 for the SConv path: per-slice accumulators acc = W x slice (the microkernel
 * of algos.py:328-330) for a slice range; layouts as described at cb_slice_plan. */
int cb_sconv_gemm(int variant, const cb_conv_desc* d, const cb_slice_plan* plan,
                  int32_t first_slice, int32_t count, const float* slices, const void* w_hi,
                  const void* w_lo, const float* w_f32, float* acc, void* stream);

/* ---- K5: unpack a slice range's accumulators into NCHW y, with bias
 * (algos.py:331-333; bias is the _alloc_output initialisation, algos.py:87-96). */
int cb_unpack_f32(const cb_conv_desc* d, const cb_slice_plan* plan, int32_t first_slice,
                  int32_t count, const float* acc, const float* bias, float* y, void* stream);

/* ---- K6/K7: fused implicit-GEMM convolution from NCHW: y = conv(x, w) + bias.
 * Replaces conv_baseline_im2col_gemm / conv_main_blocked_direct as a whole
 * (algos.py:185-209, :265-334).
 *
 * Tensor-core variants run one of two paths, chosen per descriptor (cb_fused_layout):
 *   path 1 (TMA): K0 splits x once into an NHWC (hi, lo) workspace, K6 is a persistent
 *          tcgen05 kernel fed by TMA im2col loads of that workspace and tiled TMA loads of
 *          the tap-ordered split weights;
 *   path 0 (gather): no workspace; producer warps gather + split from NCHW (used when TMA
 *          im2col cannot express the descriptor, e.g. groups not chunk aligned).
 * FFMA always runs the SIMT gather kernel with raw OIHW weights (no packing). */
typedef struct cb_fused_layout {
    int32_t path;            /* 1 = TMA im2col, 0 = gather                                  */
    int32_t chunk_channels;  /* channels per reduction chunk (path 1)                      */
    int32_t chunk_bytes;     /* 16 / 32 / 64 / 128 (path 1)                                */
    int32_t k_blocks;        /* pipeline stages per output tile                            */
    int32_t weight_rows;     /* packed weight matrix: rows (= out_channels) ...            */
    int32_t weight_cols;     /* ... x cols elements per half (0 for FFMA: raw OIHW)        */
    int64_t workspace_bytes; /* activation split workspace (0 unless path 1)               */
} cb_fused_layout;

int cb_fused_layout_query(int variant, const cb_conv_desc* d, cb_fused_layout* layout);

/* Reduction layout of the direct few-channel path (path 2, K7): the packed weight rows and
 * the kernel's A operand order the reduction as map[k] = (c * k_h + r) * k_w + s, the OIHW
 * offset of the tap at position k, or -1 for a zero element (pad taps).  Writes min(*kdim,
 * capacity) entries; *kdim is the layout's length before rounding to weight_cols.
 * CB_ERR_UNSUPPORTED for the other paths.  Host arithmetic only. */
int cb_fused_reduction_map(int variant, const cb_conv_desc* d, int32_t capacity, int32_t* map,
                           int32_t* kdim);

/* Tile plan of cb_conv_fused_packed (the persistent grid for path 1). */
int cb_fused_plan_tiles(int variant, const cb_conv_desc* d, cb_tile_plan* plan);

/* K3 for the fused path (PRE_REORDER): OIHW weights -> packed split halves in the layout
 * the selected path consumes (weight_rows x weight_cols each; bf16 halves as uint16). */
int cb_fused_pack_weights(int variant, const cb_conv_desc* d, const float* w, void* w_hi,
                          void* w_lo, void* stream);

/* K0 (IN_PACKING): x -> NHWC (hi, lo) split in `workspace` (no-op unless path 1). */
int cb_fused_pack_input(int variant, const cb_conv_desc* d, const float* x, void* workspace,
                        size_t workspace_bytes, void* stream);

/* K6/K7 (IN_MICROKERNEL) on already packed operands.
 *
 * Concurrency contract: when the tile plan splits the tail tiles along K (cb_fused_plan_tiles
 * reports it through the workspace size), the K parts of a tile wait for one another across
 * CTAs, so every CTA of the persistent grid (at most one per SM) must be resident at once.
 * The library checks the grid against the occupancy API of an idle device
 * (CB_ERR_UNSUPPORTED otherwise).  Do not run this call concurrently with other kernels on
 * other streams of the same GPU, or under an MPS SM cap: stream-ordered use -- every
 * kernel of this library, one stream per process -- is the supported mode. */
int cb_conv_fused_packed(int variant, const cb_conv_desc* d, const float* x,
                         const void* workspace, size_t workspace_bytes, const void* w_hi,
                         const void* w_lo, const float* w_f32, const float* bias, float* y,
                         void* stream);

/* K0 + K6 in one call (weights already packed by cb_fused_pack_weights). */
int cb_conv_fused(int variant, const cb_conv_desc* d, const float* x, const void* w_hi,
                  const void* w_lo, const float* w_f32, const float* bias, float* y,
                  void* workspace, size_t workspace_bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* CONVB200_H */
