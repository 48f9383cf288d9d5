// capi.cu -- extern "C" entry points of libconvb200.so (declared in include/convb200.h).
//
// Validation mirrors the reference's data-model checks (ConvDescriptor.__post_init__,
// descriptor.py:45-59; output_shape, descriptor.py:84-92; ConvInputs shape checks,
// algos.py:47-59) so that status codes map 1:1 onto the reference exception types.
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include <unistd.h>  // environ

#include "cb_common.cuh"

namespace cb {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }
int fail(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}
static std::atomic<uint64_t> g_launches{0};

int check_launch(const char* what) {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess)
        return fail(CB_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
    return CB_OK;
}

static thread_local std::vector<const char*> t_env;  // "CB_X=value" strings of environ
static thread_local bool t_env_ready = false;

void env_refresh() {
    t_env.clear();
    for (char** e = environ; e && *e; ++e)
        if ((*e)[0] == 'C' && (*e)[1] == 'B' && (*e)[2] == '_') t_env.push_back(*e);
    t_env_ready = true;
}

const char* env(const char* name) {
    if (!t_env_ready) env_refresh();
    const size_t n = std::strlen(name);
    for (const char* e : t_env)
        if (std::strncmp(e, name, n) == 0 && e[n] == '=') return e + n + 1;
    return nullptr;
}

int promote_k(bool bf16) {  // read per launch: a host-side getenv; tests toggle it in-process
    const char* e = env("CB_PROMOTE_K");
    const int v = e ? std::atoi(e) : bf16 ? 4096 : 2048;
    return v > 0 ? v : (1 << 30);
}

int sm_count() {
    static int count = 0;
    static std::once_flag once;
    std::call_once(once, [] {
        int dev = 0, n = 0;
        if (cudaGetDevice(&dev) == cudaSuccess &&
            cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess)
            count = n;
        else
            count = 148;
    });
    return count;
}

int make_geom(const cb_conv_desc* d, Geom* g) {
    env_refresh();  // one environment scan per C-ABI call (cb_common.cuh: env)
    if (!d) return fail(CB_ERR_INVALID, "null descriptor");
    const int32_t pos[] = {d->batch, d->in_channels, d->in_h, d->in_w, d->out_channels, d->k_h,
                           d->k_w, d->stride_h, d->stride_w, d->dil_h, d->dil_w, d->groups};
    const char* names[] = {"batch", "in_channels", "in_h", "in_w", "out_channels", "k_h",
                           "k_w", "stride_h", "stride_w", "dil_h", "dil_w", "groups"};
    for (int i = 0; i < 12; ++i)
        if (pos[i] < 1)
            return fail(CB_ERR_INVALID,
                        std::string(names[i]) + " must be >= 1, got " + std::to_string(pos[i]));
    if (d->pad_h < 0 || d->pad_w < 0) return fail(CB_ERR_INVALID, "padding must be >= 0");
    if (d->in_channels % d->groups)
        return fail(CB_ERR_INVALID, "in_channels not divisible by groups");
    if (d->out_channels % d->groups)
        return fail(CB_ERR_INVALID, "out_channels not divisible by groups");
    if (d->has_bias != 0 && d->has_bias != 1) return fail(CB_ERR_INVALID, "has_bias must be 0/1");
    const int64_t P = ((int64_t)d->in_h + 2LL * d->pad_h - (int64_t)d->dil_h * (d->k_h - 1) - 1) /
                          d->stride_h + 1;
    const int64_t Q = ((int64_t)d->in_w + 2LL * d->pad_w - (int64_t)d->dil_w * (d->k_w - 1) - 1) /
                          d->stride_w + 1;
    if (P < 1 || Q < 1)
        return fail(CB_ERR_INVALID, "kernel does not fit: output would be " + std::to_string(P) +
                                        "x" + std::to_string(Q));
    Geom& o = *g;
    o.N = d->batch;
    o.C = d->in_channels;
    o.H = d->in_h;
    o.W = d->in_w;
    o.K = d->out_channels;
    o.R = d->k_h;
    o.S = d->k_w;
    o.sh = d->stride_h;
    o.sw = d->stride_w;
    o.ph = d->pad_h;
    o.pw = d->pad_w;
    o.dh = d->dil_h;
    o.dw = d->dil_w;
    o.G = d->groups;
    o.P = (int)P;
    o.Q = (int)Q;
    o.cpg = o.C / o.G;
    o.kpg = o.K / o.G;
    const int64_t kdim = (int64_t)o.cpg * o.R * o.S;
    if (kdim > (1 << 30)) return fail(CB_ERR_UNSUPPORTED, "reduction too long");
    o.kdim = (int)kdim;
    o.kdim_pad = cb_split_kdim(o.kdim);
    o.PQ = o.P * o.Q;
    o.HW = o.H * o.W;
    o.RS = o.R * o.S;
    o.npix = (int64_t)o.N * o.PQ;
    return CB_OK;
}

int launch_im2col_band(const Geom& g, const float* x, float* out, bool sliced, int band_rows,
                       int first_slice, int count, int64_t j_begin, int64_t j_count,
                       cudaStream_t st);
int launch_im2col(const Geom& g, const float* x, float* out, int64_t j_begin, int64_t j_count,
                  cudaStream_t st);
int launch_weight_split(bool bf16, int rows, int kdim, int kdim_pad, const float* w, void* hi,
                        void* lo, cudaStream_t st);
int launch_unpack(const Geom& g, int band_rows, int64_t j_begin, int64_t j_count,
                  const float* acc, const float* bias, float* y, cudaStream_t st);
int tc_plan_query(const Geom& g, int64_t npix, bool bf16, bool allow_split, cb_tile_plan* out);
int tma_plan_query(const Geom& g, bool bf16, cb_tile_plan* out);
FusedLayout fused_layout(const Geom& g, bool bf16);
int launch_act_split(bool bf16, const Geom& g, int c_alloc, const float* x, void* hi, void* lo,
                     int* counters, int n_counters, cudaStream_t st, int fold);
int launch_weight_split_taps(bool bf16, const Geom& g, int CB, int chk, int kw_pad, const float* w,
                             void* hi, void* lo, cudaStream_t st, int fold, int stack_rs,
                             int k_orig);
int launch_tap_sum(const Geom& g, int mode, const float* yp, const float* bias, float* y,
                   cudaStream_t st);
int launch_conv_tma(bool bf16, const Geom& g, const FusedLayout& L, const void* act_hi,
                    const void* act_lo, const void* w_hi, const void* w_lo, const float* bias,
                    float* y, void* tail_ws, cudaStream_t st);
int64_t tma_tail_workspace_bytes(const Geom& g, const FusedLayout& L);
int debug_trace_copy(unsigned long long* host, int max_ctas, int* slots);
int tma_tail_counters(const Geom& g, const FusedLayout& L);
int launch_conv_ts(const Geom& g, bool bf16, const float* x, const void* w_hi, const void* w_lo,
                   const float* bias, float* y, cudaStream_t st);
int ts_plan_query(const Geom& g, bool bf16, cb_tile_plan* out);
int ts_reduction_map(const Geom& g, bool bf16, int cap, int32_t* map);
int ts_weight_kdim(const Geom& g, bool bf16, int* pair, int* pf);
int launch_weight_split_pairs(const Geom& g, bool bf16, int pf, int kdim_pad, int mixed, const float* w,
                              void* hi, void* lo, cudaStream_t st);
int ffma_plan_query(const Geom& g, int64_t npix, bool allow_split, cb_tile_plan* out);
int launch_tc(bool bf16, const Geom& g, const PixMap& pm, const float* src, const void* w_hi,
              const void* w_lo, const float* bias, float* out, int add_mode, int zero_kind,
              cudaStream_t st);
int launch_ffma(const Geom& g, const PixMap& pm, const float* src, const float* w,
                const float* bias, float* out, int add_mode, int zero_kind, cudaStream_t st);

int launch_gemm_ts(bool bf16, const Geom& g, const PixMap& pm, const float* src, const void* w_hi,
                   const void* w_lo, const float* bias, float* out, int add_mode, cudaStream_t st);

static int run_variant(int variant, const Geom& g, const PixMap& pm, const float* src,
                       const void* w_hi, const void* w_lo, const float* w_f32, const float* bias,
                       float* out, int add_mode, int zero_kind, cudaStream_t st) {
    switch (variant) {
        case CB_VARIANT_TC3XTF32:
        case CB_VARIANT_TC3XBF16:
            if (!w_hi || !w_lo) return fail(CB_ERR_INVALID, "tensor-core variants need split weights");
            {  // K8 (A in TMEM) for the matrix / slice GEMMs; K4 otherwise
                const int rc = launch_gemm_ts(variant == CB_VARIANT_TC3XBF16, g, pm, src, w_hi,
                                              w_lo, bias, out, add_mode, st);
                if (rc != CB_ERR_UNSUPPORTED) return rc;
            }
            return launch_tc(variant == CB_VARIANT_TC3XBF16, g, pm, src, w_hi, w_lo, bias, out,
                             add_mode, zero_kind, st);
        case CB_VARIANT_FFMA:
            if (!w_f32) return fail(CB_ERR_INVALID, "FFMA variant needs raw fp32 weights");
            return launch_ffma(g, pm, src, w_f32, bias, out, add_mode, zero_kind, st);
        default:
            return fail(CB_ERR_UNSUPPORTED, "unknown variant " + std::to_string(variant));
    }
}

static int check_plan(const Geom& g, const cb_slice_plan* plan) {
    if (!plan) return fail(CB_ERR_INVALID, "null slice plan");
    if (plan->band_rows < 1) return fail(CB_ERR_INVALID, "band_rows must be >= 1");
    const int64_t want = (int64_t)g.N * ((g.P + plan->band_rows - 1) / plan->band_rows);
    if (plan->num_slices != want) return fail(CB_ERR_INVALID, "slice plan does not match descriptor");
    return CB_OK;
}

// pixel range of slices [first, first+count)
static int slice_range(const Geom& g, const cb_slice_plan* plan, int32_t first, int32_t count,
                       int64_t* jb, int64_t* jc) {
    if (first < 0 || count < 0 || (int64_t)first + count > plan->num_slices)
        return fail(CB_ERR_INVALID, "slice range outside the plan");
    const int64_t b = slice_pixel_begin(g, plan->band_rows, first);
    const int64_t e = slice_pixel_begin(g, plan->band_rows, (int64_t)first + count);
    *jb = b;
    *jc = e - b;
    return CB_OK;
}

static PixMap full_range(const Geom& g) {
    PixMap pm{};
    pm.j_begin = 0;
    pm.j_count = g.npix;
    return pm;
}

static int sconv_supported(const Geom& g) {
    // blocked direct rejects grouped / dilated descriptors (algos.py:277-280)
    if (g.G != 1 || g.dh != 1 || g.dw != 1)
        return fail(CB_ERR_UNSUPPORTED,
                    "blocked direct requires groups == 1 and dilation == 1, got groups=" +
                        std::to_string(g.G) + ", dilation=(" + std::to_string(g.dh) + ", " +
                        std::to_string(g.dw) + ")");
    return CB_OK;
}

}  // namespace cb

using namespace cb;

extern "C" {

int cb_version(void) { return CB_ABI_VERSION; }

const char* cb_last_error_string(void) { return cb::g_last_error.c_str(); }

uint64_t cb_launch_count(void) { return cb::g_launches.load(std::memory_order_relaxed); }

// Diagnostics (not in convb200.h): per-CTA globaltimer stamps of the latest fused-conv
// launch made with CB_TMA_TRACE set.  Returns the CTA count copied.
int cb_debug_trace(unsigned long long* host, int max_ctas, int* slots) {
    return cb::debug_trace_copy(host, max_ctas, slots);
}

int cb_event_create(void** ev) {
    if (!ev) return fail(CB_ERR_INVALID, "null out pointer");
    cudaEvent_t e = nullptr;
    cudaError_t rc = cudaEventCreateWithFlags(&e, cudaEventDefault);
    if (rc != cudaSuccess) return fail(CB_ERR_CUDA, std::string("cudaEventCreate: ") + cudaGetErrorString(rc));
    *ev = e;
    return CB_OK;
}

int cb_event_destroy(void* ev) {
    if (ev) cudaEventDestroy(static_cast<cudaEvent_t>(ev));
    return CB_OK;
}

int cb_event_record(void* ev, void* stream, int external) {
    if (!ev) return fail(CB_ERR_INVALID, "null event");
    cudaError_t rc = cudaEventRecordWithFlags(static_cast<cudaEvent_t>(ev),
                                              static_cast<cudaStream_t>(stream),
                                              external ? cudaEventRecordExternal : cudaEventRecordDefault);
    if (rc != cudaSuccess) return fail(CB_ERR_CUDA, std::string("cudaEventRecord: ") + cudaGetErrorString(rc));
    return CB_OK;
}

int cb_event_elapsed_ns(void* e0, void* e1, int64_t* ns) {
    if (!e0 || !e1 || !ns) return fail(CB_ERR_INVALID, "null argument");
    cudaError_t rc = cudaEventSynchronize(static_cast<cudaEvent_t>(e1));
    float ms = 0.f;
    if (rc == cudaSuccess)
        rc = cudaEventElapsedTime(&ms, static_cast<cudaEvent_t>(e0), static_cast<cudaEvent_t>(e1));
    if (rc != cudaSuccess) return fail(CB_ERR_CUDA, std::string("cudaEventElapsedTime: ") + cudaGetErrorString(rc));
    *ns = (int64_t)llround((double)ms * 1e6);
    return CB_OK;
}

int cb_device_sm_count(int* n) {
    if (!n) return fail(CB_ERR_INVALID, "null out pointer");
    *n = sm_count();
    return CB_OK;
}

uint64_t cb_env_fingerprint(void) {
    uint64_t h = 1469598103934665603ULL;  // FNV-1a over every "CB_name=value" string, in order
    for (char** e = environ; e && *e; ++e) {
        if ((*e)[0] != 'C' || (*e)[1] != 'B' || (*e)[2] != '_') continue;
        for (const char* c = *e; *c; ++c) h = (h ^ (unsigned char)*c) * 1099511628211ULL;
        h = (h ^ 0xffu) * 1099511628211ULL;
    }
    return h;
}

int cb_output_shape(const cb_conv_desc* d, int32_t* oh, int32_t* ow) {
    Geom g;
    int rc = make_geom(d, &g);
    if (rc) return rc;
    if (oh) *oh = g.P;
    if (ow) *ow = g.Q;
    return CB_OK;
}

int32_t cb_split_kdim(int32_t kdim) { return kdim <= 0 ? 0 : (kdim + 63) / 64 * 64; }

int cb_workspace_bytes(const cb_conv_desc* d, int algo, const cb_slice_plan* plan, size_t* bytes) {
    Geom g;
    int rc = make_geom(d, &g);
    if (rc) return rc;
    if (!bytes) return fail(CB_ERR_INVALID, "null out pointer");
    switch (algo) {
        case 0: *bytes = (size_t)g.C * g.RS * g.npix * sizeof(float); return CB_OK;
        case 1:
            if ((rc = sconv_supported(g))) return rc;
            if ((rc = check_plan(g, plan))) return rc;
            *bytes = ((size_t)g.kdim + g.K) * g.npix * sizeof(float);
            return CB_OK;
        case 2: *bytes = 0; return CB_OK;
        default: return fail(CB_ERR_INVALID, "unknown algorithm id " + std::to_string(algo));
    }
}

int cb_im2col_f32(const cb_conv_desc* d, const float* x, float* cols, void* stream) {
    Geom g;
    int rc = make_geom(d, &g);
    if (rc) return rc;
    if (!x || !cols) return fail(CB_ERR_INVALID, "null buffer");
    // smem-staged band kernel; the per-element kernel covers windows too wide for smem
    rc = launch_im2col_band(g, x, cols, false, 0, 0, 0, 0, g.npix, (cudaStream_t)stream);
    if (rc != CB_ERR_UNSUPPORTED) return rc;
    return launch_im2col(g, x, cols, 0, g.npix, (cudaStream_t)stream);
}

int cb_sconv_plan(const cb_conv_desc* d, int32_t max_slice_pixels, cb_slice_plan* plan) {
    Geom g;
    int rc = make_geom(d, &g);
    if (rc) return rc;
    if ((rc = sconv_supported(g))) return rc;
    if (!plan) return fail(CB_ERR_INVALID, "null plan");
    int band = max_slice_pixels / g.Q;
    band = band < 1 ? 1 : (band > g.P ? g.P : band);
    plan->band_rows = band;
    plan->num_slices = g.N * ((g.P + band - 1) / band);
    return CB_OK;
}

int cb_sconv_range(const cb_conv_desc* d, const cb_slice_plan* plan, int32_t first_slice,
                   int32_t count, int64_t* pix_begin, int64_t* pix_count) {
    Geom g;
    int rc = make_geom(d, &g);
    if (rc) return rc;
    if ((rc = check_plan(g, plan))) return rc;
    if (!pix_begin || !pix_count) return fail(CB_ERR_INVALID, "null out pointer");
    return slice_range(g, plan, first_slice, count, pix_begin, pix_count);
}

int cb_sconv_pack_f32(const cb_conv_desc* d, const cb_slice_plan* plan, int32_t first_slice,
                      int32_t count, const float* x, float* slices, void* stream) {
    Geom g;
    int rc = make_geom(d, &g);
    if (rc) return rc;
    if ((rc = sconv_supported(g)) || (rc = check_plan(g, plan))) return rc;
    if (!x || !slices) return fail(CB_ERR_INVALID, "null buffer");
    int64_t jb, jc;
    if ((rc = slice_range(g, plan, first_slice, count, &jb, &jc))) return rc;
    if (count == 0) return CB_OK;
    rc = launch_im2col_band(g, x, slices, true, plan->band_rows, first_slice, count, jb, jc,
                            (cudaStream_t)stream);
    if (rc != CB_ERR_UNSUPPORTED) return rc;
    return launch_im2col(g, x, slices, jb, jc, (cudaStream_t)stream);
}

int cb_plan_tiles(int variant, const cb_conv_desc* d, int64_t pixels, cb_tile_plan* plan) {
    Geom g;
    int rc = make_geom(d, &g);
    if (rc) return rc;
    if (!plan) return fail(CB_ERR_INVALID, "null out pointer");
    const int64_t np = pixels <= 0 ? g.npix : pixels;
    switch (variant) {
        case CB_VARIANT_TC3XTF32:
        case CB_VARIANT_TC3XBF16:
            return tc_plan_query(g, np, variant == CB_VARIANT_TC3XBF16, true, plan);
        case CB_VARIANT_FFMA: return ffma_plan_query(g, np, true, plan);
        default: return fail(CB_ERR_UNSUPPORTED, "unknown variant " + std::to_string(variant));
    }
}

int cb_weight_split(int variant, int32_t rows, int32_t kdim, const float* w, void* w_hi,
                    void* w_lo, void* stream) {
    if (rows < 0 || kdim < 0) return fail(CB_ERR_INVALID, "negative weight shape");
    if (!w || !w_hi || !w_lo) return fail(CB_ERR_INVALID, "null buffer");
    if (variant != CB_VARIANT_TC3XTF32 && variant != CB_VARIANT_TC3XBF16)
        return fail(CB_ERR_INVALID, "weight split is only defined for the tensor-core variants");
    return launch_weight_split(variant == CB_VARIANT_TC3XBF16, rows, kdim, cb_split_kdim(kdim), w,
                               w_hi, w_lo, (cudaStream_t)stream);
}

int cb_gemm(int variant, int32_t m, int32_t n, int32_t k, const void* a_hi, const void* a_lo,
            const float* a_f32, const float* b, int64_t ldb, float* c, int64_t ldc,
            int accumulate, void* stream) {
    env_refresh();
    if (m < 0 || n < 0 || k < 0) return fail(CB_ERR_INVALID, "negative GEMM shape");
    if (ldb < n || ldc < n) return fail(CB_ERR_INVALID, "leading dimension smaller than n");
    if (m == 0 || n == 0) return CB_OK;
    if (!b || !c) return fail(CB_ERR_INVALID, "null buffer");
    Geom g{};
    g.N = 1;
    g.R = g.S = g.RS = 1;
    g.K = m;
    g.G = 1;
    g.kpg = m;
    g.kdim = k;
    g.kdim_pad = cb_split_kdim(k);
    g.npix = n;
    g.PQ = n;
    g.P = 1;
    g.Q = n;
    PixMap pm = full_range(g);
    pm.src_mode = SRC_MATRIX;
    pm.dst_mode = DST_MATRIX;
    pm.src_ld = ldb;
    pm.dst_ld = ldc;
    if (k == 0) {
        if (accumulate) return CB_OK;
        // c = 0 (empty reduction): reuse the kernel with a zero-length k loop is not
        // possible, so clear row by row.
        for (int32_t i = 0; i < m; ++i) {
            cudaError_t e = cudaMemsetAsync(c + (int64_t)i * ldc, 0, sizeof(float) * n,
                                            (cudaStream_t)stream);
            if (e != cudaSuccess) return fail(CB_ERR_CUDA, cudaGetErrorString(e));
        }
        return CB_OK;
    }
    return run_variant(variant, g, pm, b, a_hi, a_lo, a_f32, nullptr, c, accumulate ? 1 : 0,
                       /*zero_kind=*/0, (cudaStream_t)stream);
}

int cb_conv_gemm_cols(int variant, const cb_conv_desc* d, const float* cols, const void* w_hi,
                      const void* w_lo, const float* w_f32, const float* bias, float* y,
                      void* stream) {
    Geom g;
    int rc = make_geom(d, &g);
    if (rc) return rc;
    if (!cols || !y) return fail(CB_ERR_INVALID, "null buffer");
    if (d->has_bias && !bias) return fail(CB_ERR_INVALID, "descriptor has bias but bias is null");
    PixMap pm = full_range(g);
    pm.src_mode = SRC_MATRIX;
    pm.src_ld = g.npix;
    pm.dst_mode = DST_NCHW;
    return run_variant(variant, g, pm, cols, w_hi, w_lo, w_f32, d->has_bias ? bias : nullptr, y,
                       0, /*zero_kind=NCHW bias fill*/ 1, (cudaStream_t)stream);
}

int cb_sconv_gemm(int variant, const cb_conv_desc* d, const cb_slice_plan* plan,
                  int32_t first_slice, int32_t count, const float* slices, const void* w_hi,
                  const void* w_lo, const float* w_f32, float* acc, void* stream) {
    Geom g;
    int rc = make_geom(d, &g);
    if (rc) return rc;
    if ((rc = sconv_supported(g)) || (rc = check_plan(g, plan))) return rc;
    if (!slices || !acc) return fail(CB_ERR_INVALID, "null buffer");
    int64_t jb, jc;
    if ((rc = slice_range(g, plan, first_slice, count, &jb, &jc))) return rc;
    // the chunk's slice buffer is the (kdim x jc) im2col matrix of its pixels and the
    // accumulators a (K x jc) matrix: a plain GEMM over launch-local pixels, whose tiles
    // run across slice boundaries
    PixMap pm{};
    pm.src_mode = SRC_MATRIX;
    pm.dst_mode = DST_MATRIX;
    pm.src_ld = jc;
    pm.dst_ld = jc;
    pm.j_begin = 0;
    pm.j_count = jc;
    return run_variant(variant, g, pm, slices, w_hi, w_lo, w_f32, nullptr, acc, 0,
                       /*zero_kind=contiguous memset*/ 2, (cudaStream_t)stream);
}

int cb_unpack_f32(const cb_conv_desc* d, const cb_slice_plan* plan, int32_t first_slice,
                  int32_t count, const float* acc, const float* bias, float* y, void* stream) {
    Geom g;
    int rc = make_geom(d, &g);
    if (rc) return rc;
    if ((rc = sconv_supported(g)) || (rc = check_plan(g, plan))) return rc;
    if (!acc || !y) return fail(CB_ERR_INVALID, "null buffer");
    if (d->has_bias && !bias) return fail(CB_ERR_INVALID, "descriptor has bias but bias is null");
    int64_t jb, jc;
    if ((rc = slice_range(g, plan, first_slice, count, &jb, &jc))) return rc;
    return launch_unpack(g, plan->band_rows, jb, jc, acc, d->has_bias ? bias : nullptr, y,
                         (cudaStream_t)stream);
}

// g: the descriptor's geometry (K0 reads x with it); gk: the geometry the TMA kernel, its
// plan and the weight pack run on -- fold_geom(g) when the layout folds, else g.
static int fused_setup(int variant, const cb_conv_desc* d, Geom* g, FusedLayout* L,
                       Geom* gk = nullptr) {
    int rc = make_geom(d, g);
    if (rc) return rc;
    if (variant != CB_VARIANT_TC3XTF32 && variant != CB_VARIANT_TC3XBF16 &&
        variant != CB_VARIANT_FFMA)
        return fail(CB_ERR_UNSUPPORTED, "unknown variant " + std::to_string(variant));
    *L = FusedLayout{};
    if (variant != CB_VARIANT_FFMA) *L = fused_layout(*g, variant == CB_VARIANT_TC3XBF16);
    if (gk) *gk = L->stack ? stack_geom(*g, L->stack) : L->fold ? fold_geom(*g) : *g;
    return CB_OK;
}

// Fused workspace = [act hi | act lo | tail split-K counters + partials], 256-B aligned parts.
static void act_halves(const FusedLayout& L, void* ws, void** hi, void** lo, void** tail) {
    const size_t half = ((size_t)L.act_elems * L.eb + 255) / 256 * 256;
    *hi = ws;
    *lo = static_cast<uint8_t*>(ws) + half;
    *tail = static_cast<uint8_t*>(ws) + 2 * half;
}

static int64_t act_ws_bytes(const Geom& g, const FusedLayout& L) {
    if (!L.tma) return 0;
    const int64_t tail = (tma_tail_workspace_bytes(g, L) + 255) / 256 * 256;
    // stacked taps: + the 1x1 conv's output Y' (fp32 NCHW over the input grid)
    const int64_t stacked = L.stack ? (int64_t)g.N * g.K * g.PQ * 4 : 0;
    return 2 * (((int64_t)L.act_elems * L.eb + 255) / 256 * 256) + tail + stacked;
}
static float* stack_buffer(const Geom& gk, const FusedLayout& L, void* ws) {
    const int64_t tail = (tma_tail_workspace_bytes(gk, L) + 255) / 256 * 256;
    return reinterpret_cast<float*>(static_cast<uint8_t*>(ws) +
                                    2 * (((int64_t)L.act_elems * L.eb + 255) / 256 * 256) + tail);
}

int cb_fused_layout_query(int variant, const cb_conv_desc* d, cb_fused_layout* out) {
    Geom g, gk;
    FusedLayout L;
    int rc = fused_setup(variant, d, &g, &L, &gk);
    if (rc) return rc;
    if (!out) return fail(CB_ERR_INVALID, "null out pointer");
    *out = cb_fused_layout{};
    out->weight_rows = gk.K;  // stacked taps: R*S*K rows
    if (variant == CB_VARIANT_FFMA) {
        out->path = 0;
        out->k_blocks = (g.kdim + 15) / 16;
        return CB_OK;
    }
    out->path = L.ts ? 2 : L.tma;
    out->chunk_channels = L.tma ? L.cb : 0;
    out->chunk_bytes = L.tma ? L.chunk_bytes : 0;
    out->k_blocks = L.tma ? L.num_kb : (g.kdim + 128 / L.eb - 1) / (128 / L.eb);
    int ts_pair = 0, ts_pf = 0;
    out->weight_cols = L.tma ? L.kw_pad
                             : cb_split_kdim(L.ts ? ts_weight_kdim(g, variant == CB_VARIANT_TC3XBF16, &ts_pair, &ts_pf) : g.kdim);  // K7 / K4
    out->workspace_bytes = act_ws_bytes(gk, L);
    return CB_OK;
}

int cb_fused_reduction_map(int variant, const cb_conv_desc* d, int32_t capacity, int32_t* map,
                           int32_t* kdim) {
    Geom g, gk;
    FusedLayout L;
    int rc = fused_setup(variant, d, &g, &L, &gk);
    if (rc) return rc;
    if (!kdim || (capacity > 0 && !map)) return fail(CB_ERR_INVALID, "null out pointer");
    if (variant == CB_VARIANT_FFMA || !L.ts)
        return fail(CB_ERR_UNSUPPORTED, "only the direct few-channel path (path 2) has a reduction map");
    const int kd = ts_reduction_map(g, variant == CB_VARIANT_TC3XBF16, capacity, map);
    if (kd < 0) return fail(CB_ERR_UNSUPPORTED, "direct TMEM conv does not fit this descriptor");
    *kdim = kd;
    return CB_OK;
}

int cb_fused_plan_tiles(int variant, const cb_conv_desc* d, cb_tile_plan* plan) {
    Geom g, gk;
    FusedLayout L;
    int rc = fused_setup(variant, d, &g, &L, &gk);
    if (rc) return rc;
    if (!plan) return fail(CB_ERR_INVALID, "null out pointer");
    if (variant == CB_VARIANT_FFMA) return ffma_plan_query(g, g.npix, true, plan);
    if (L.ts) return ts_plan_query(g, variant == CB_VARIANT_TC3XBF16, plan);
    if (L.tma) return tma_plan_query(gk, variant == CB_VARIANT_TC3XBF16, plan);
    return tc_plan_query(g, g.npix, variant == CB_VARIANT_TC3XBF16, true, plan);
}

int cb_fused_pack_weights(int variant, const cb_conv_desc* d, const float* w, void* w_hi,
                          void* w_lo, void* stream) {
    Geom g, gk;
    FusedLayout L;
    int rc = fused_setup(variant, d, &g, &L, &gk);
    if (rc) return rc;
    if (variant == CB_VARIANT_FFMA)
        return fail(CB_ERR_INVALID, "the FFMA variant consumes raw OIHW weights");
    if (!w || !w_hi || !w_lo) return fail(CB_ERR_INVALID, "null buffer");
    const bool bf16 = variant == CB_VARIANT_TC3XBF16;
    if (L.tma)
        return launch_weight_split_taps(bf16, gk, L.cb, L.chk, L.kw_pad, w, w_hi, w_lo,
                                        (cudaStream_t)stream, L.fold,
                                        L.stack == 1 ? g.RS : L.stack == 2 ? g.S : 0, g.K);
    if (L.ts) {  // K7: plain split rows, or the pair layout with one pad tap per (c, r) row
        int pair = 0, pf = 0;
        const int kd = ts_weight_kdim(g, bf16, &pair, &pf);
        if (pair) return launch_weight_split_pairs(g, bf16, pf, cb_split_kdim(kd), pair == 2, w, w_hi, w_lo, (cudaStream_t)stream);
    }
    return launch_weight_split(bf16, g.K, g.kdim, cb_split_kdim(g.kdim), w, w_hi, w_lo,
                               (cudaStream_t)stream);
}

int cb_fused_pack_input(int variant, const cb_conv_desc* d, const float* x, void* ws,
                        size_t ws_bytes, void* stream) {
    Geom g, gk;
    FusedLayout L;
    int rc = fused_setup(variant, d, &g, &L, &gk);
    if (rc) return rc;
    if (variant == CB_VARIANT_FFMA || !L.tma) return CB_OK;
    if (!x || !ws) return fail(CB_ERR_INVALID, "null buffer");
    if ((int64_t)ws_bytes < act_ws_bytes(gk, L))
        return fail(CB_ERR_WORKSPACE, "workspace too small: need " +
                                          std::to_string(act_ws_bytes(gk, L)) + " bytes");
    void *hi, *lo, *tail;
    act_halves(L, ws, &hi, &lo, &tail);
    return launch_act_split(variant == CB_VARIANT_TC3XBF16, g, L.c_alloc, x, hi, lo,
                            static_cast<int*>(tail), tma_tail_counters(gk, L), (cudaStream_t)stream,
                            L.fold);
}

int cb_conv_fused_packed(int variant, const cb_conv_desc* d, const float* x, const void* ws,
                         size_t ws_bytes, const void* w_hi, const void* w_lo, const float* w_f32,
                         const float* bias, float* y, void* stream) {
    Geom g, gk;
    FusedLayout L;
    int rc = fused_setup(variant, d, &g, &L, &gk);
    if (rc) return rc;
    if (!y) return fail(CB_ERR_INVALID, "null output");
    if (d->has_bias && !bias) return fail(CB_ERR_INVALID, "descriptor has bias but bias is null");
    const float* b = d->has_bias ? bias : nullptr;
    if (variant != CB_VARIANT_FFMA && L.ts) {
        if (!x) return fail(CB_ERR_INVALID, "null input");
        if (!w_hi || !w_lo) return fail(CB_ERR_INVALID, "tensor-core variants need packed weights");
        return launch_conv_ts(g, variant == CB_VARIANT_TC3XBF16, x, w_hi, w_lo, b, y, (cudaStream_t)stream);
    }
    if (variant != CB_VARIANT_FFMA && L.tma) {
        if (!ws || (int64_t)ws_bytes < act_ws_bytes(gk, L))
            return fail(CB_ERR_WORKSPACE, "workspace too small: need " +
                                              std::to_string(act_ws_bytes(gk, L)) + " bytes");
        if (!w_hi || !w_lo) return fail(CB_ERR_INVALID, "tensor-core variants need packed weights");
        void *hi, *lo, *tail;
        act_halves(L, const_cast<void*>(ws), &hi, &lo, &tail);
        if (L.stack) {  // 1x1 conv into Y', then K9 sums the shifted taps (+bias) into y
            float* yp = stack_buffer(gk, L, const_cast<void*>(ws));
            rc = launch_conv_tma(variant == CB_VARIANT_TC3XBF16, gk, L, hi, lo, w_hi, w_lo, nullptr,
                                 yp, tail, (cudaStream_t)stream);
            if (rc) return rc;
            return launch_tap_sum(g, L.stack, yp, b, y, (cudaStream_t)stream);
        }
        return launch_conv_tma(variant == CB_VARIANT_TC3XBF16, gk, L, hi, lo, w_hi, w_lo, b, y, tail,
                               (cudaStream_t)stream);
    }
    if (!x) return fail(CB_ERR_INVALID, "null input");
    PixMap pm = full_range(g);
    pm.src_mode = SRC_CONV;
    pm.dst_mode = DST_NCHW;
    return run_variant(variant, g, pm, x, w_hi, w_lo, w_f32, b, y, 0,
                       /*zero_kind=NCHW bias fill*/ 1, (cudaStream_t)stream);
}

int cb_conv_fused(int variant, const cb_conv_desc* d, const float* x, const void* w_hi,
                  const void* w_lo, const float* w_f32, const float* bias, float* y, void* ws,
                  size_t ws_bytes, void* stream) {
    int rc = cb_fused_pack_input(variant, d, x, ws, ws_bytes, stream);
    if (rc) return rc;
    return cb_conv_fused_packed(variant, d, x, ws, ws_bytes, w_hi, w_lo, w_f32, bias, y, stream);
}

}  // extern "C"
