// pack_kernels.cu -- the HBM-bound packing kernels of the two stepwise algorithms.
//
//   K1 im2col_kernel<false>  im2col_transform        (algos.py:99-121)   -> PRE_REORDER
//   K2 im2col_kernel<true>   SConv per-slice packing (algos.py:305-324)  -> IN_PACKING
//   K3 weight_split_kernel   wmat / _pack_a_panels   (algos.py:124-130, :202, :291)
//   K5 unpack_kernel         out[...] += acc         (algos.py:331-333)  -> IN_UNPACKING
//   fill_bias_kernel         _alloc_output           (algos.py:87-96)
//
// K1/K2 are pure copies (bit-exact with the reference): each thread owns VEC
// consecutive output columns (pixels) of one packed row (c, ky, kx), so stores are
// coalesced 16-byte vectors and the loads of a warp walk one input row.  The input is
// read through L2 once from HBM (every tap re-reads it from L2); the packed matrix is
// written once: algorithmic bytes = 4 * (N*C*H*W + C*R*S*N*P*Q).
#include <algorithm>

#include <cudaTypedefs.h>

#include <mutex>

#include "cb_common.cuh"
#include "sm100_ptx.cuh"

namespace cb {

constexpr int PACK_VEC = 4;
constexpr int PACK_THREADS = 256;

__global__ void __launch_bounds__(PACK_THREADS)
im2col_kernel(Geom g, const float* __restrict__ x, float* __restrict__ out, int64_t j_begin,
              int64_t j_count, int64_t col_blocks, bool vec_ok) {
    const int64_t bid = blockIdx.x;
    const int row = (int)(bid / col_blocks);
    const int64_t cblk = bid - (int64_t)row * col_blocks;
    const int64_t jl = (cblk * PACK_THREADS + threadIdx.x) * PACK_VEC;
    if (jl >= j_count) return;
    const int64_t j = j_begin + jl;

    // row = (c, ky, kx) over ALL input channels (groups are contiguous row blocks)
    const int c = row / g.RS;
    const int rs = row - c * g.RS;
    const int ky = rs / g.S;
    const int kx = rs - ky * g.S;

    int64_t n = j / g.PQ;
    int p = (int)(j - n * g.PQ);
    int oy = p / g.Q;
    int ox = p - oy * g.Q;

    float v[PACK_VEC];
#pragma unroll
    for (int i = 0; i < PACK_VEC; ++i) {
        float val = 0.f;
        if (jl + i < j_count) {
            const int iy = oy * g.sh - g.ph + ky * g.dh;
            const int ix = ox * g.sw - g.pw + kx * g.dw;
            if ((unsigned)iy < (unsigned)g.H && (unsigned)ix < (unsigned)g.W)
                val = __ldg(x + (((int64_t)n * g.C + c) * g.H + iy) * g.W + ix);
        }
        v[i] = val;
        if (++ox == g.Q) {
            ox = 0;
            if (++oy == g.P) {
                oy = 0;
                ++n;
            }
        }
    }

    // (k, pixel) with row stride j_count: the im2col columns (K1) or a chunk's slices (K2)
    float* dst = out + (int64_t)row * j_count + jl;
    if (vec_ok) {
        *reinterpret_cast<float4*>(dst) = make_float4(v[0], v[1], v[2], v[3]);
    } else {
#pragma unroll
        for (int i = 0; i < PACK_VEC; ++i)
            if (jl + i < j_count) dst[i] = v[i];
    }
}

// ---------------------------------------------------------------------------------------
// K1/K2 (band kernel): one block = (image n, CC channels, a band of TR output rows).
// The zero-padded input window of the band -- IR = (TR-1)*sh + (R-1)*dh + 1 rows of
// W + 2*pw columns per channel -- is staged in smem with coalesced row reads (each input
// element read from L2 once per block instead of once per tap), then every (c, ky, kx)
// packed row of the band is written as one contiguous run of TR*Q pixels: one LDS and one
// coalesced STG per output element.  The kernel is HBM-write bound.
//   SLICED = false: dst = cols[row][j]                   (im2col_transform layout)
//   SLICED = true : dst = slices[row][j - j_begin] of the chunk's (kdim x j_count) matrix
//                   (blocks walk the chunk's slices; a band never crosses a slice)
// ---------------------------------------------------------------------------------------
constexpr int BAND_THREADS = 256;
constexpr int BAND_MAXM = 8;  // pixels per band <= BAND_THREADS * BAND_MAXM

struct BandPlan {
    int TR;            // output rows per band
    int CC;            // channels per block
    int IR, IWp;       // staged window rows / row pitch
    int bands_per_unit;  // bands per image (K1) or per slice (K2)
    int PXT;             // pixels of a full band (offset-table size)
    // TMA staging: the window is one 4-D box {IWp, IR, CC, 1} of x loaded at column -x0
    // (x0 = pw rounded up to 4: 16-byte aligned start), zero-filled outside the tensor;
    // window column = input column + x0.  0: per-element loads, column = input col + pw.
    int tma, x0;
    // NB > 1 (K1 with TMA, whole-image bands of small images): a block packs NB consecutive
    // images -- one box {IWp, IR, CC, NB} -- so each packed row run is NB * P * Q pixels
    int NB;
    size_t smem;
};

template <bool SLICED>
__global__ void __launch_bounds__(BAND_THREADS)
im2col_band_kernel(Geom g, BandPlan bp, const float* __restrict__ x, float* __restrict__ out,
                   int band_rows, int first_slice, int64_t j_begin, int64_t j_count,
                   const __grid_constant__ CUtensorMap tm_x) {
    extern __shared__ __align__(128) float smem_band[];  // [CC][IR][IWp][pixel tab][row tab]
    __shared__ __align__(8) uint64_t win_bar;
    float* win = smem_band;
    int* off_tab = reinterpret_cast<int*>(smem_band + (size_t)bp.NB * bp.CC * bp.IR * bp.IWp);
    // ---- which band ----
    const int unit = blockIdx.x / bp.bands_per_unit;  // image (K1) or slice index (K2)
    const int sub = blockIdx.x - unit * bp.bands_per_unit;
    int n, y_lo, y_hi;  // output rows [y_lo, y_hi) of image n
    int nb = 1;  // images of this block (NB > 1: whole-image bands, y_lo = 0)
    if (!SLICED) {
        n = unit * bp.NB;
        nb = min(bp.NB, g.N - n);
        y_lo = sub * bp.TR;
        y_hi = min(g.P, y_lo + bp.TR);
    } else {
        const int per_img = (g.P + band_rows - 1) / band_rows;
        const int s = first_slice + unit;
        n = s / per_img;
        const int s0 = (s - n * per_img) * band_rows;
        const int s1 = min(g.P, s0 + band_rows);
        y_lo = s0 + sub * bp.TR;
        y_hi = min(s1, y_lo + bp.TR);
    }
    if (y_lo >= y_hi) return;  // block-uniform
    const int c0 = blockIdx.y * bp.CC;
    const int cc = min(bp.CC, g.C - c0);
    const int npx = nb * (y_hi - y_lo) * g.Q;
    const int iy0 = y_lo * g.sh - g.ph;
    const int ir = (y_hi - y_lo - 1) * g.sh + (g.R - 1) * g.dh + 1;
    // ---- stage the zero-padded window [cc][ir][IWp] (this band's own row count, so the
    //      smem index of element e is e); (c, r, col) advance by counters, no division ----
    const float* xb = x + ((int64_t)n * g.C + c0) * g.HW;
    const int tot = cc * ir * bp.IWp;
    const int wrows = bp.tma ? bp.IR : ir;  // window plane rows (the TMA box is always full)
    if (bp.tma) {
        if (threadIdx.x == 0) {
            ptx::mbar_init(&win_bar, 1);
            ptx::fence_mbar_init();
            ptx::mbar_arrive_expect_tx(&win_bar, (uint32_t)(bp.NB * bp.CC * bp.IR * bp.IWp * 4));
            ptx::tma_load_4d(win, &tm_x, &win_bar, -bp.x0, iy0, c0, n);  // NB images: box dim 3
        }
    } else {
        const int plane = ir * bp.IWp;
        // BAND_THREADS in the mixed radix (c, r, col) = (., ir, IWp)
        const int drow = BAND_THREADS / bp.IWp, dcol = BAND_THREADS - drow * bp.IWp;
        const int dc = drow / ir, dr = drow - dc * ir;
        int e = threadIdx.x;
        int c = e / plane;
        int r = (e - c * plane) / bp.IWp;
        int col = e - c * plane - r * bp.IWp;
        while (e < tot) {
            float v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int iy = iy0 + r, ix = col - g.pw;
                v[u] = 0.f;
                if (e + u * BAND_THREADS < tot && (unsigned)iy < (unsigned)g.H &&
                    (unsigned)ix < (unsigned)g.W)
                    v[u] = __ldg(xb + (int64_t)c * g.HW + iy * g.W + ix);
                col += dcol;
                r += dr;
                c += dc;
                if (col >= bp.IWp) { col -= bp.IWp; ++r; }
                if (r >= ir) { r -= ir; ++c; }
            }
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (e + u * BAND_THREADS < tot) win[e + u * BAND_THREADS] = v[u];
            e += 8 * BAND_THREADS;
        }
    }
    // ---- pixel -> window offset table (the same for every packed row of the band) and
    //      packed row -> window base table (no integer division in the store loop) ----
    int* row_tab = off_tab + (bp.PXT + 3) / 4 * 4;
    const int col0 = bp.tma ? bp.x0 - g.pw : 0;  // window column of the band's first tap
    const int bpx = (y_hi - y_lo) * g.Q;                   // pixels per image of the band
    const int img_words = bp.CC * bp.IR * bp.IWp;          // window words per image (NB > 1)
    for (int pix = threadIdx.x; pix < npx; pix += BAND_THREADS) {
        const int b = bp.NB > 1 ? pix / bpx : 0;
        const int pl = pix - b * bpx;
        const int oyl = pl / g.Q;
        off_tab[pix] = b * img_words + oyl * g.sh * bp.IWp + (pl - oyl * g.Q) * g.sw + col0;
    }
    const int nrows = cc * g.RS;
    for (int r = threadIdx.x; r < nrows; r += BAND_THREADS) {
        const int c = r / g.RS;
        const int t = r - c * g.RS;
        const int ky = t / g.S, kx = t - (t / g.S) * g.S;
        row_tab[r] = (c * wrows + ky * g.dh) * bp.IWp + kx * g.dw;
    }
    __syncthreads();
    if (bp.tma) ptx::mbar_wait(&win_bar, 0);
    // ---- destination of this band's run in every packed row ----
    const int64_t row_stride = j_count;
    const int64_t dst0 = (int64_t)n * g.PQ + (int64_t)y_lo * g.Q - j_begin;
    // ---- each warp streams 4 packed rows (c, ky, kx) per pass; one offset-table load
    //      feeds 4 gathers and 4 coalesced stores ----
    constexpr int NW = BAND_THREADS / 32;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float* const out_b = out + dst0 + (int64_t)c0 * g.RS * row_stride;
    for (int r0 = warp * 4; r0 < nrows; r0 += 4 * NW) {
        const int nr = min(4, nrows - r0);  // warp-uniform
        const float* w0 = win + row_tab[r0];
        const float* w1 = win + row_tab[min(r0 + 1, nrows - 1)];
        const float* w2 = win + row_tab[min(r0 + 2, nrows - 1)];
        const float* w3 = win + row_tab[min(r0 + 3, nrows - 1)];
        float* d0 = out_b + (int64_t)r0 * row_stride;
        float* d1 = d0 + row_stride;
        float* d2 = d1 + row_stride;
        float* d3 = d2 + row_stride;
        if (nr == 4) {
#pragma unroll 2
            for (int pix = lane; pix < npx; pix += 32) {
                const int o = off_tab[pix];
                const float v0 = w0[o], v1 = w1[o], v2 = w2[o], v3 = w3[o];
                d0[pix] = v0;
                d1[pix] = v1;
                d2[pix] = v2;
                d3[pix] = v3;
            }
        } else {
            for (int pix = lane; pix < npx; pix += 32) {
                const int o = off_tab[pix];
                d0[pix] = w0[o];
                if (nr > 1) d1[pix] = w1[o];
                if (nr > 2) d2[pix] = w2[o];
            }
        }
    }
}

// Band geometry: ~1-2K pixels per band (<= BAND_THREADS * BAND_MAXM), window <= 40 KB.
static bool band_plan(const Geom& g, int max_rows, int64_t units, BandPlan* bp, bool multi_image) {
    const int cap_px = BAND_THREADS * BAND_MAXM;
    if (g.Q > cap_px) return false;
    int tr = std::max(1, std::min(max_rows, 1536 / std::max(1, g.Q)));
    tr = std::min(tr, std::max(1, cap_px / g.Q));
    auto per_ch_of = [&](int t) {
        return (size_t)((t - 1) * g.sh + (g.R - 1) * g.dh + 1) * (g.W + 2 * g.pw) * sizeof(float);
    };
    // ~16 KB windows keep ~8 blocks (64 warps) resident per SM, so one block's staging
    // loads overlap the other blocks' streaming stores
    int cc = (int)std::max<size_t>(1, std::min<size_t>(g.C, (16 * 1024) / per_ch_of(tr)));
    // at least ~2 waves of blocks: shrink the channel group, then the band (>= 256 px)
    static const int waves = [] {
        const char* e = getenv("CB_BAND_WAVES");
        return e ? atoi(e) : 2;  // with the TMA-staged window: cfg4 K1 59 -> 50 us (0: off)
    }();
    const int64_t want = (int64_t)waves * sm_count() * 8;
    auto blocks = [&](int t, int c) {
        return units * ((max_rows + t - 1) / t) * ((g.C + c - 1) / c);
    };
    while (blocks(tr, cc) < want && cc > 1) cc = (cc + 1) / 2;
    // (bands are not shrunk by default: smaller bands measured slower -- cfg2b 8.4 -> 10.5 us)
    static const bool shrink_bands = getenv("CB_BAND_SHRINK_ROWS") != nullptr;
    while (shrink_bands && blocks(tr, cc) < want && tr > 1 && (tr / 2) * g.Q >= 256) tr /= 2;
    bp->TR = tr;
    bp->IR = (tr - 1) * g.sh + (g.R - 1) * g.dh + 1;
    bp->IWp = g.W + 2 * g.pw;
    bp->tma = 0;
    bp->x0 = 0;
    {
        const int x0 = (g.pw + 3) / 4 * 4;
        const int bw = (g.W + g.pw + x0 + 3) / 4 * 4;
        static const bool no_tma = getenv("CB_BAND_NO_TMA") != nullptr;
        if (!no_tma && g.W % 4 == 0 && bw <= 256 && bp->IR <= 256 && cc <= 256) {
            bp->tma = 1;
            bp->x0 = x0;
            bp->IWp = bw;
        }
    }
    const size_t per_ch = (size_t)bp->IR * bp->IWp * sizeof(float);
    if (per_ch > 96 * 1024) return false;
    bp->NB = 1;
    // (measured neutral on cfg4, so off unless CB_BAND_NB is set)
    static const bool use_nb = getenv("CB_BAND_NB") != nullptr;
    if (multi_image && use_nb && bp->tma && tr == max_rows && g.PQ < 1024 && g.N > 1) {
        // runs of >= ~1K pixels; the window budget is shared by the NB images
        bp->NB = (int)std::min<int64_t>(std::min(g.N, 256), (1024 + g.PQ - 1) / g.PQ);
        cc = (int)std::max<size_t>(1, std::min<size_t>(cc, (16 * 1024) / (per_ch * bp->NB)));
    }
    bp->CC = cc;
    bp->PXT = bp->NB * tr * g.Q;  // offset-table entries (pixels of a full band)
    bp->smem = per_ch * bp->CC * bp->NB + sizeof(int) * ((bp->PXT + 3) / 4 * 4) +
               sizeof(int) * (size_t)bp->CC * g.RS;
    if (bp->smem > 200 * 1024) {  // (tiny channel groups never get here)
        bp->tma = 0;
        bp->NB = 1;
    }
    return true;
}

int launch_im2col_band(const Geom& g, const float* x, float* out, bool sliced, int band_rows,
                       int first_slice, int count, int64_t j_begin, int64_t j_count,
                       cudaStream_t st) {
    BandPlan bp{};
    const int64_t units = sliced ? count : g.N;
    if (!band_plan(g, sliced ? band_rows : g.P, units, &bp, !sliced)) return CB_ERR_UNSUPPORTED;
    bp.bands_per_unit = ((sliced ? band_rows : g.P) + bp.TR - 1) / bp.TR;
    const int64_t gx = (units + bp.NB - 1) / bp.NB * bp.bands_per_unit;
    const int64_t gy = (g.C + bp.CC - 1) / bp.CC;
    if (gx > 0x7fffffffLL || gy > 65535) return CB_ERR_UNSUPPORTED;
    CUtensorMap tm{};
    if (bp.tma && (reinterpret_cast<uintptr_t>(x) & 15)) bp.tma = 0;
    if (bp.tma) {
        static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
        static std::once_flag once;
        std::call_once(once, [] {
            void* ptr = nullptr;
            cudaDriverEntryPointQueryResult q;
            if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
                    cudaSuccess && q == cudaDriverEntryPointSuccess)
                enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
        });
        cuuint64_t dims[4] = {(cuuint64_t)g.W, (cuuint64_t)g.H, (cuuint64_t)g.C, (cuuint64_t)g.N};
        cuuint64_t strides[3] = {(cuuint64_t)g.W * 4, (cuuint64_t)g.HW * 4, (cuuint64_t)g.C * g.HW * 4};
        cuuint32_t box[4] = {(cuuint32_t)bp.IWp, (cuuint32_t)bp.IR, (cuuint32_t)bp.CC, (cuuint32_t)bp.NB};
        cuuint32_t es[4] = {1, 1, 1, 1};
        if (!enc || enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(x), dims, strides,
                        box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return fail(CB_ERR_CUDA, "cuTensorMapEncodeTiled (band window) failed");
    }
    auto kern = sliced ? im2col_band_kernel<true> : im2col_band_kernel<false>;
    if (bp.smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)bp.smem);
        if (e != cudaSuccess) return fail(CB_ERR_CUDA, cudaGetErrorString(e));
    }
    kern<<<dim3((unsigned)gx, (unsigned)gy), BAND_THREADS, bp.smem, st>>>(
        g, bp, x, out, band_rows, first_slice, j_begin, j_count, tm);
    return check_launch(sliced ? "sconv_pack_band" : "im2col_band");
}

// K3: rows x kdim (row-major) -> hi/lo rows x kdim_pad, zero padded.
template <bool BF16>
__global__ void weight_split_kernel(int rows, int kdim, int kdim_pad, const float* __restrict__ w,
                                    void* __restrict__ hi_out, void* __restrict__ lo_out) {
    // rows by blockIdx.y, columns by a block-stride loop: no 64-bit division per element
    for (int r = blockIdx.y; r < rows; r += gridDim.y)
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < kdim_pad; k += gridDim.x * blockDim.x) {
        const int64_t i = (int64_t)r * kdim_pad + k;
        const float v = k < kdim ? w[(int64_t)r * kdim + k] : 0.f;
        if (BF16) {
            const uint16_t h = bf16_rn_bits(v);
            const uint16_t l = bf16_rn_bits(v - bf16_bits_to_f32(h));
            static_cast<uint16_t*>(hi_out)[i] = h;
            static_cast<uint16_t*>(lo_out)[i] = l;
        } else {
            const Split2 s = split_tf32(v);
            static_cast<float*>(hi_out)[i] = s.hi;
            static_cast<float*>(lo_out)[i] = s.lo;
        }
    }
}

// y (N, K, P*Q) = bias broadcast (or 0): the output initialisation of _alloc_output.
__global__ void fill_bias_kernel(int64_t images, int K, int PQ, const float* __restrict__ bias,
                                 float* __restrict__ y) {
    const int64_t total = images * K * PQ;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int f = (int)((i / PQ) % K);
        y[i] = bias ? __ldg(bias + f) : 0.f;
    }
}

static int grid_for(int64_t total, int threads) {
    const int64_t want = ceil_div64(total, threads);
    const int64_t cap = (int64_t)sm_count() * 16;
    return (int)(want < cap ? (want > 0 ? want : 1) : cap);
}

int launch_im2col(const Geom& g, const float* x, float* out, int64_t j_begin, int64_t j_count,
                  cudaStream_t st) {
    if (j_count == 0) return CB_OK;
    const int64_t col_blocks = ceil_div64(j_count, (int64_t)PACK_THREADS * PACK_VEC);
    const int64_t rows = (int64_t)g.C * g.RS;
    const int64_t blocks = rows * col_blocks;
    if (blocks > 0x7fffffffLL) return fail(CB_ERR_UNSUPPORTED, "im2col grid too large");
    const bool vec_ok = (reinterpret_cast<uintptr_t>(out) & 15) == 0 && (j_count % PACK_VEC == 0);
    im2col_kernel<<<(unsigned)blocks, PACK_THREADS, 0, st>>>(g, x, out, j_begin, j_count,
                                                             col_blocks, vec_ok);
    return check_launch(j_begin || j_count != g.npix ? "sconv_pack" : "im2col");
}

int launch_weight_split(bool bf16, int rows, int kdim, int kdim_pad, const float* w, void* hi,
                        void* lo, cudaStream_t st) {
    const int64_t total = (int64_t)rows * kdim_pad;
    if (total == 0) return CB_OK;
    const dim3 grid((unsigned)std::min<int64_t>((kdim_pad + 255) / 256, 16), (unsigned)std::min(rows, 65535));
    if (bf16)
        weight_split_kernel<true><<<grid, 256, 0, st>>>(rows, kdim, kdim_pad, w, hi, lo);
    else
        weight_split_kernel<false><<<grid, 256, 0, st>>>(rows, kdim, kdim_pad, w, hi, lo);
    return check_launch("weight_split");
}

// K3 for K7's pair layout: rows K x kdim_pad, k = (c*R + r)*(S+1) + s', the pad tap s' = 0
// (pf = 1) or s' = S (pf = 0) zero, split into bf16 (hi, lo).
template <bool BF16>
__global__ void weight_split_pairs_kernel(int K, int C, int R, int S, int pf, int kdim_pad, int mixed,
                                          const float* __restrict__ w, void* __restrict__ hi_out,
                                          void* __restrict__ lo_out) {
    const int f = blockIdx.y;
    const int SP = S + 1, KD = C * R * SP;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < kdim_pad; k += gridDim.x * blockDim.x) {
        float v = 0.f;
        if (mixed) {  // the K7 mixed layout (cb_common.cuh: mixed_map)
            const MixedTap t = mixed_map(k, C * R, S, pf);
            if (t.cr >= 0) v = w[((int64_t)f * C + t.cr / R) * R * S + (t.cr % R) * S + t.s];
        } else if (k < KD) {
            const int cr = k / SP, s = k - cr * SP - pf;
            if (s >= 0 && s < S) v = w[((int64_t)f * C + cr / R) * R * S + (cr % R) * S + s];
        }
        if (BF16) {
            const uint16_t h = bf16_rn_bits(v);
            static_cast<uint16_t*>(hi_out)[(int64_t)f * kdim_pad + k] = h;
            static_cast<uint16_t*>(lo_out)[(int64_t)f * kdim_pad + k] = bf16_rn_bits(v - bf16_bits_to_f32(h));
        } else {
            const Split2 sp = split_tf32(v);
            static_cast<float*>(hi_out)[(int64_t)f * kdim_pad + k] = sp.hi;
            static_cast<float*>(lo_out)[(int64_t)f * kdim_pad + k] = sp.lo;
        }
    }
}

int launch_weight_split_pairs(const Geom& g, bool bf16, int pf, int kdim_pad, int mixed, const float* w,
                              void* hi, void* lo, cudaStream_t st) {
    if (g.K == 0) return CB_OK;
    if (g.K > 65535) return fail(CB_ERR_UNSUPPORTED, "too many output channels for weight pack");
    const dim3 grid((unsigned)((kdim_pad + 255) / 256), (unsigned)g.K);
    if (bf16)
        weight_split_pairs_kernel<true><<<grid, 256, 0, st>>>(g.K, g.C, g.R, g.S, pf, kdim_pad, mixed, w, hi, lo);
    else
        weight_split_pairs_kernel<false><<<grid, 256, 0, st>>>(g.K, g.C, g.R, g.S, pf, kdim_pad, mixed, w, hi, lo);
    return check_launch("weight_split_pairs");
}

// K5 by rows: a slice is a band of whole output rows of one image, so each (slice, channel)
// pair is one contiguous run in both the accumulator matrix and y.  One warp per run, float4
// when both ends are 16-byte aligned.
__global__ void __launch_bounds__(256)
unpack_rows_kernel(Geom g, int band_rows, int64_t s_first, int64_t j_begin, int64_t j_count,
                   int64_t nrows, const float* __restrict__ acc, const float* __restrict__ bias,
                   float* __restrict__ y) {
    const int64_t row = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (row >= nrows) return;
    const int64_t ls = row / g.K;
    const int f = (int)(row - ls * g.K);
    const int per_img = (g.P + band_rows - 1) / band_rows;
    const int64_t sg = s_first + ls;
    const int64_t n = sg / per_img;
    const int y0 = (int)(sg - n * per_img) * band_rows;
    const int np = min(band_rows, g.P - y0) * g.Q;
    const int64_t j0 = n * g.PQ + (int64_t)y0 * g.Q;
    const float* src = acc + (int64_t)f * j_count + (j0 - j_begin);
    float* dst = y + (n * g.K + f) * g.PQ + (int64_t)y0 * g.Q;
    const float b = bias ? __ldg(bias + f) : 0.f;
    if (((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0) {
        const int n4 = np >> 2;
        const float4* s4 = reinterpret_cast<const float4*>(src);
        float4* d4 = reinterpret_cast<float4*>(dst);
        // 8 vectors in flight per lane (the loop was latency-bound at one)
        int i = lane;
        for (; i + 224 < n4; i += 256) {
            float4 v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = __ldg(s4 + i + 32 * u);
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                v[u].x += b; v[u].y += b; v[u].z += b; v[u].w += b;
                d4[i + 32 * u] = v[u];
            }
        }
        for (; i + 96 < n4; i += 128) {
            float4 v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) v[u] = __ldg(s4 + i + 32 * u);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                v[u].x += b; v[u].y += b; v[u].z += b; v[u].w += b;
                d4[i + 32 * u] = v[u];
            }
        }
        for (; i < n4; i += 32) {
            float4 v = __ldg(s4 + i);
            v.x += b; v.y += b; v.z += b; v.w += b;
            d4[i] = v;
        }
        for (int i = (n4 << 2) + lane; i < np; i += 32) dst[i] = __ldg(src + i) + b;
    } else {
        for (int i = lane; i < np; i += 32) dst[i] = __ldg(src + i) + b;
    }
}

// K5 when every slice is a whole image (band_rows >= P): image i of the chunk is the
// column block acc[:, i*PQ : (i+1)*PQ] of the K x J accumulator matrix and y's images are
// contiguous, so y is walked linearly in float4 lanes, 4 vectors in flight per thread; each
// vector's (image, channel, pixel) advances by the grid stride in mixed radix (no division
// in the loop).
__global__ void __launch_bounds__(256)
unpack_images_kernel(int64_t nvec, int pq4, int K, int64_t j4, const float4* __restrict__ acc,
                     const float* __restrict__ bias, float4* __restrict__ y) {
    const int64_t stride = (int64_t)gridDim.x * 256;
    const int64_t img4 = (int64_t)K * pq4;
    // the stride and this thread's first vector in (image, channel, pixel) digits
    const int64_t s_im = stride / img4;
    const int s_f = (int)((stride - s_im * img4) / pq4);
    const int s_p = (int)(stride - s_im * img4 - (int64_t)s_f * pq4);
    int64_t i = blockIdx.x * 256LL + threadIdx.x;
    int64_t im = i / img4;
    int f = (int)((i - im * img4) / pq4);
    int p = (int)(i - im * img4 - (int64_t)f * pq4);
    auto advance = [&] {
        i += stride;
        p += s_p;
        f += s_f;
        im += s_im;
        if (p >= pq4) { p -= pq4; ++f; }
        if (f >= K) { f -= K; ++im; }
    };
    while (i < nvec) {
        float4 v[4];
        int fu[4];
        int64_t iu[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            iu[u] = i;
            fu[u] = f;
            if (i < nvec) v[u] = __ldcs(acc + (int64_t)f * j4 + im * pq4 + p);
            advance();
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            if (iu[u] >= nvec) break;
            if (bias) {
                const float b = __ldg(bias + fu[u]);
                v[u].x += b, v[u].y += b, v[u].z += b, v[u].w += b;
            }
            y[iu[u]] = v[u];
        }
    }
}

int launch_unpack(const Geom& g, int band_rows, int64_t j_begin, int64_t j_count,
                  const float* acc, const float* bias, float* y, cudaStream_t st) {
    const int64_t total = j_count * g.K;
    if (total == 0) return CB_OK;
    if (band_rows >= g.P && g.PQ % 4 == 0 && j_begin % g.PQ == 0 && j_count % g.PQ == 0 &&
        ((reinterpret_cast<uintptr_t>(acc) | reinterpret_cast<uintptr_t>(y)) & 15) == 0 &&
        !env("CB_K5_ROWS")) {
        const int64_t nvec = total / 4;
        const int64_t blocks = std::min<int64_t>((nvec + 1023) / 1024, (int64_t)sm_count() * 8);
        unpack_images_kernel<<<(unsigned)std::max<int64_t>(1, blocks), 256, 0, st>>>(
            nvec, g.PQ / 4, g.K, j_count / 4, reinterpret_cast<const float4*>(acc), bias,
            reinterpret_cast<float4*>(y + (j_begin / g.PQ) * (int64_t)g.K * g.PQ));
        return check_launch("unpack_images");
    }
    // the launch covers whole slices: count them from the first slice's index
    const int per_img = (g.P + band_rows - 1) / band_rows;
    const int64_t n0 = j_begin / g.PQ;
    const int oy0 = (int)((j_begin - n0 * g.PQ) / g.Q);
    const int64_t s_first = n0 * per_img + oy0 / band_rows;
    int64_t nslices = 0;
    for (int64_t j = j_begin; j < j_begin + j_count; ++nslices) {
        const int64_t sg = s_first + nslices;
        const int64_t n = sg / per_img;
        const int y0 = (int)(sg - n * per_img) * band_rows;
        j = n * g.PQ + (int64_t)y0 * g.Q + (int64_t)std::min(band_rows, g.P - y0) * g.Q;
    }
    const int64_t nrows = nslices * g.K;
    const int64_t blocks = (nrows + 7) / 8;
    if (blocks > 0x7fffffffLL) return fail(CB_ERR_UNSUPPORTED, "unpack grid too large");
    unpack_rows_kernel<<<(unsigned)blocks, 256, 0, st>>>(g, band_rows, s_first, j_begin, j_count,
                                                          nrows, acc, bias, y);
    return check_launch("unpack");
}

int launch_fill_bias(int64_t images, int K, int PQ, const float* bias, float* y, cudaStream_t st) {
    const int64_t total = images * K * PQ;
    if (total == 0) return CB_OK;
    fill_bias_kernel<<<grid_for(total, 256), 256, 0, st>>>(images, K, PQ, bias, y);
    return check_launch("fill_bias");
}

// ---------------------------------------------------------------------------------------
// K0: activation split + NCHW -> NHWC reorder for the TMA-fed fused conv.
// Every input element is split exactly once (hi = rn(x), lo = rn(x - hi)) and written
// channel-innermost with a c_alloc pitch (zero padded), the layout TMA im2col mode walks.
// 32 x 32 (pixel x channel) smem-transposed tiles: reads coalesced along H*W, writes
// coalesced along the contiguous (pixel, channel) run of the tile.
// ---------------------------------------------------------------------------------------
// Splits VEC consecutive values and stores both halves as one 16-byte vector each.
template <bool BF16, int VEC>
__device__ __forceinline__ void store_split16(void* hi_out, void* lo_out, int64_t o,
                                              const float (&v)[VEC]) {
    if (BF16) {
        static_assert(!BF16 || VEC == 8, "bf16: 8 values per 16 bytes");
        uint32_t h[4], l[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const uint16_t h0 = bf16_rn_bits(v[2 * e]), h1 = bf16_rn_bits(v[2 * e + 1]);
            const uint16_t l0 = bf16_rn_bits(v[2 * e] - bf16_bits_to_f32(h0));
            const uint16_t l1 = bf16_rn_bits(v[2 * e + 1] - bf16_bits_to_f32(h1));
            h[e] = (uint32_t)h0 | ((uint32_t)h1 << 16);
            l[e] = (uint32_t)l0 | ((uint32_t)l1 << 16);
        }
        *reinterpret_cast<uint4*>(static_cast<uint16_t*>(hi_out) + o) = make_uint4(h[0], h[1], h[2], h[3]);
        *reinterpret_cast<uint4*>(static_cast<uint16_t*>(lo_out) + o) = make_uint4(l[0], l[1], l[2], l[3]);
    } else {
        static_assert(BF16 || VEC == 4, "tf32: 4 values per 16 bytes");
        float h[4], l[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const Split2 s = split_tf32(v[e]);
            h[e] = s.hi;
            l[e] = s.lo;
        }
        *reinterpret_cast<float4*>(static_cast<float*>(hi_out) + o) = make_float4(h[0], h[1], h[2], h[3]);
        *reinterpret_cast<float4*>(static_cast<float*>(lo_out) + o) = make_float4(l[0], l[1], l[2], l[3]);
    }
}

// 32 pixels x 64 channels per block: coalesced 128-byte reads along H*W into smem, then
// each thread splits one 16-byte run of channels of one pixel (c_alloc is a multiple of
// the run length) and writes hi and lo as 16-byte vectors.
template <bool BF16>
__global__ void __launch_bounds__(256)
act_split_nhwc_kernel(int C, int HW, int c_alloc, const float* __restrict__ x,
                      void* __restrict__ hi_out, void* __restrict__ lo_out, int* counters,
                      int n_counters) {
    constexpr int VEC = BF16 ? 8 : 4;
    __shared__ float tile[64][33];
    // let the dependent conv kernel (PDL) launch and run its prologue early
    asm volatile("griddepcontrol.launch_dependents;");
    // the fused conv's tail split-K counters start every launch at zero
    if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0)
        for (int i = threadIdx.x; i < n_counters; i += 256) counters[i] = 0;
    const int p0 = blockIdx.x * 32;
    const int c0 = blockIdx.y * 64;
    const int64_t n = blockIdx.z;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const float* xn = x + n * (int64_t)C * HW;
    const int p = p0 + tx;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int c = c0 + ty + 8 * i;
        tile[ty + 8 * i][tx] = (c < C && p < HW) ? __ldg(xn + (int64_t)c * HW + p) : 0.f;
    }
    __syncthreads();
    const int cw = min(64, c_alloc - c0);
    const int nq = cw / VEC;
    const int pw = min(32, HW - p0);
    const int64_t obase = (n * HW + p0) * (int64_t)c_alloc + c0;
    if (BF16 && nq == 8) {
        // one (pixel, 8-channel group) per thread, no division; paired bf16x2 conversions
        const int pix = threadIdx.x >> 3, q = threadIdx.x & 7;
        if (pix < pw) {
            uint32_t h[4], l[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const float a = tile[q * 8 + 2 * e][pix], b = tile[q * 8 + 2 * e + 1][pix];
                uint32_t hb;
                asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(hb) : "f"(b), "f"(a));
                const float ra = a - __uint_as_float(hb << 16), rb = b - __uint_as_float(hb & 0xffff0000u);
                uint32_t lb;
                asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(lb) : "f"(rb), "f"(ra));
                h[e] = hb;
                l[e] = lb;
            }
            const int64_t o = obase + (int64_t)pix * c_alloc + q * 8;
            *reinterpret_cast<uint4*>(static_cast<uint16_t*>(hi_out) + o) = make_uint4(h[0], h[1], h[2], h[3]);
            *reinterpret_cast<uint4*>(static_cast<uint16_t*>(lo_out) + o) = make_uint4(l[0], l[1], l[2], l[3]);
        }
        asm volatile("griddepcontrol.wait;" ::: "memory");  // the packing before us (K3) is complete
        return;
    }
    for (int e = threadIdx.x; e < 32 * nq; e += 256) {
        const int pix = e / nq, q = e - pix * nq;
        if (pix >= pw) break;
        float v[VEC];
#pragma unroll
        for (int j = 0; j < VEC; ++j) v[j] = tile[q * VEC + j][pix];
        store_split16<BF16, VEC>(hi_out, lo_out, obase + (int64_t)pix * c_alloc + q * VEC, v);
    }
    asm volatile("griddepcontrol.wait;" ::: "memory");  // the packing before us (K3) is complete
}

// K0, wide variant (bf16, HW % 4 == 0, 64-channel groups): a block splits 128 consecutive
// pixels of the flattened (n, p) index x 64 channels -- float4 loads of 4-pixel groups (a
// warp reads 512 contiguous bytes of a channel row), no partly empty pixel blocks.
constexpr int AS_PX = 128;
// tile[ch][px] with the 4-pixel groups of row ch XOR-swizzled by ch / 8: the float4 row
// writes stay contiguous and the transposed reads (8 channel groups x 4 pixels per warp)
// hit 32 distinct banks
__device__ __forceinline__ int as_idx(int ch, int px) {
    return ch * AS_PX + ((((px >> 2) ^ (ch >> 3)) & 31) << 2) + (px & 3);
}
__global__ void __launch_bounds__(256)
act_split_wide_kernel(int C, int HW, int64_t npix, int c_alloc, const float* __restrict__ x,
                      void* __restrict__ hi_out, void* __restrict__ lo_out, int* counters,
                      int n_counters) {
    __shared__ __align__(16) float tile[64 * AS_PX];
    asm volatile("griddepcontrol.launch_dependents;");
    if (blockIdx.x == 0 && blockIdx.y == 0)
        for (int i = threadIdx.x; i < n_counters; i += 256) counters[i] = 0;
    const int64_t j0 = (int64_t)blockIdx.x * AS_PX;
    const int c0 = blockIdx.y * 64;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t jg = j0 + 4 * lane;
    const bool gvalid = jg < npix;
    const int64_t n = gvalid ? jg / HW : 0;
    const float* xg = x + n * (int64_t)C * HW + (jg - n * HW);
    float4 v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int c = c0 + warp + 8 * i;
        v[i] = (gvalid && c < C) ? __ldg(reinterpret_cast<const float4*>(xg + (int64_t)c * HW))
                                 : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i)
        *reinterpret_cast<float4*>(tile + as_idx(warp + 8 * i, 4 * lane)) = v[i];
    __syncthreads();
    const int q = threadIdx.x & 7;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int pix = (threadIdx.x >> 3) + 32 * k;
        if (j0 + pix >= npix) break;
        uint32_t h[4], l[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const float a = tile[as_idx(q * 8 + 2 * e, pix)];
            const float b = tile[as_idx(q * 8 + 2 * e + 1, pix)];
            uint32_t hb;
            asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(hb) : "f"(b), "f"(a));
            const float ra = a - __uint_as_float(hb << 16), rb = b - __uint_as_float(hb & 0xffff0000u);
            uint32_t lb;
            asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(lb) : "f"(rb), "f"(ra));
            h[e] = hb;
            l[e] = lb;
        }
        const int64_t o = (j0 + pix) * (int64_t)c_alloc + c0 + q * 8;
        *reinterpret_cast<uint4*>(static_cast<uint16_t*>(hi_out) + o) = make_uint4(h[0], h[1], h[2], h[3]);
        *reinterpret_cast<uint4*>(static_cast<uint16_t*>(lo_out) + o) = make_uint4(l[0], l[1], l[2], l[3]);
    }
    asm volatile("griddepcontrol.wait;" ::: "memory");  // the packing before us (K3) is complete
}

// K0 for a folded layout (FusedLayout::fold): [N][H][Q][c_alloc] rows whose channel
// s*C + c holds x[n, c, ih, ox*sw + s*dw - pw] (zero outside the image and past S*C), split
// into hi / lo.  One thread per 16-byte run; the strided re-reads of x hit L1/L2.
template <bool BF16>
__global__ void __launch_bounds__(256)
act_fold_split_kernel(Geom g, int c_alloc, const float* __restrict__ x, void* __restrict__ hi_out,
                      void* __restrict__ lo_out, int* counters, int n_counters) {
    constexpr int VEC = BF16 ? 8 : 4;
    asm volatile("griddepcontrol.launch_dependents;");
    if (blockIdx.x == 0)
        for (int i = threadIdx.x; i < n_counters; i += 256) counters[i] = 0;
    const int nq = c_alloc / VEC;
    const int CS = g.C * g.S;
    const int64_t total = (int64_t)g.N * g.H * g.Q * nq;
    for (int64_t e = blockIdx.x * 256LL + threadIdx.x; e < total; e += (int64_t)gridDim.x * 256) {
        const int64_t pix = e / nq;  // (n*H + ih)*Q + ox
        const int q = (int)(e - pix * nq);
        const int64_t nh = pix / g.Q;
        const int ox = (int)(pix - nh * g.Q);
        const int64_t n = nh / g.H;
        const int ih = (int)(nh - n * g.H);
        const float* xr = x + (n * g.C * g.H + ih) * (int64_t)g.W;
        float v[VEC];
#pragma unroll
        for (int j = 0; j < VEC; ++j) {
            const int cp = q * VEC + j;
            const int s = cp / g.C, c = cp - s * g.C;
            const int ix = ox * g.sw + s * g.dw - g.pw;
            v[j] = (cp < CS && (unsigned)ix < (unsigned)g.W) ? __ldg(xr + (int64_t)c * g.HW + ix) : 0.f;
        }
        store_split16<BF16, VEC>(hi_out, lo_out, pix * c_alloc + q * VEC, v);
    }
    asm volatile("griddepcontrol.wait;" ::: "memory");  // the packing before us (K3) is complete
}

// K3 (fused layout): OIHW -> rows K x kw_pad, k = ((r*S + s)*chk + cb)*CB + ci, zero padded,
// split into hi / lo.  Matches the (tap, channel-chunk) order the TMA im2col walk feeds.
// One thread produces one 16-byte run of k (kw_pad is a multiple of 64 elements).
// Block (channel chunk of WS_CH, out channel f): the chunk's OIHW slice w[f, c0:c0+WS_CH, :, :]
// is one contiguous run, read coalesced into smem; every tap's WS_CH channels are then
// contiguous in the output row, written as 16-byte vectors.  Chunk 0 also zeroes the row
// tail [R*S*per_tap, kw_pad).
constexpr int WS_CH = 128;
template <bool BF16>
__global__ void __launch_bounds__(256)
weight_split_taps_kernel(int K, int cpg, int R, int S, int CB, int chk, int kw_pad,
                         const float* __restrict__ w, void* __restrict__ hi_out,
                         void* __restrict__ lo_out, int fold, int stack_rs, int k_orig) {
    constexpr int VEC = BF16 ? 8 : 4;
    extern __shared__ float ws_tile[];  // [WS_CH][R*S]
    // the activation split (K0) does not read the weights: it may start right away and
    // waits for this grid only at its end (griddepcontrol.wait), before the conv reads both
    asm volatile("griddepcontrol.launch_dependents;");
    const int f = blockIdx.y;
    const int c0 = blockIdx.x * WS_CH;
    const int RS = R * S;
    const int per_tap = chk * CB;
    const int nch = min(WS_CH, cpg - c0);  // real channels in this chunk (may be <= 0)
    // folded (fold = original S, S == 1 here, one chunk): stage all of w[f] in OIHW order
    // and read channel c' = s*C + c of tap r from w[f, c, r, s]
    // stacked taps (stack_rs = T > 1 taps stacked into the rows): row f = t*K + fo, kernel tap
    // tk reads the original tap tk*T + t of w[fo, c] (all R*S taps: RS = 1; the S horizontal
    // taps: RS = R, T = S)
    if (stack_rs > 1) {
        const int fo = f % k_orig, t = f / k_orig;
        const float* srcs = w + ((int64_t)fo * cpg + c0) * (RS * stack_rs) + t;
        for (int i = threadIdx.x; i < max(nch, 0) * RS; i += 256) {
            const int cl = i / RS, tk = i - cl * RS;
            ws_tile[i] = __ldg(srcs + ((int64_t)cl * RS + tk) * stack_rs);
        }
    } else {
        // the chunk is one contiguous run: 8 loads in flight per thread before any store (a
        // rolled load -> st.shared loop paid one DRAM round trip per element: 4.6 us on cfg4)
        const float* src = w + ((int64_t)f * cpg + c0) * RS;
        const int n = max(nch, 0) * RS;
        for (int i0 = 0; i0 < n; i0 += 256 * 8) {
            float v[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int i = i0 + j * 256 + threadIdx.x;
                v[j] = i < n ? __ldg(src + i) : 0.f;
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int i = i0 + j * 256 + threadIdx.x;
                if (i < n) ws_tile[i] = v[j];
            }
        }
    }
    __syncthreads();
    const int c_orig = fold ? cpg / fold : 0;
    const int cw = min(WS_CH, per_tap - c0);  // output channels of this chunk per tap
    const int nq = cw / VEC;
    const int64_t row = (int64_t)f * kw_pad;
    for (int e = threadIdx.x; e < RS * nq; e += 256) {
        const int tap = e / nq, q = e - tap * nq;
        float v[VEC];
#pragma unroll
        for (int j = 0; j < VEC; ++j) {
            const int cl = q * VEC + j;
            if (cl >= nch)
                v[j] = 0.f;
            else if (fold)
                v[j] = ws_tile[(((c0 + cl) % c_orig) * R + tap) * fold + (c0 + cl) / c_orig];
            else
                v[j] = ws_tile[cl * RS + tap];
        }
        store_split16<BF16, VEC>(hi_out, lo_out, row + (int64_t)tap * per_tap + c0 + q * VEC, v);
    }
    if (blockIdx.x == 0) {
        for (int k = RS * per_tap + threadIdx.x * VEC; k < kw_pad; k += 256 * VEC) {
            float z[VEC] = {};
            store_split16<BF16, VEC>(hi_out, lo_out, row + k, z);
        }
    }
}

// K0 launches use programmatic stream serialization: they may start while the weight split
// (K3) before them still runs (K3 triggers griddepcontrol.launch_dependents at its start; K0
// waits for it at its end), so the pair costs one launch gap instead of a fork and a join.
template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, int block, size_t smem, cudaStream_t st,
                              Args... args) {
    static const bool no_pdl = std::getenv("CB_NO_PDL") != nullptr;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = no_pdl ? 0 : 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

int launch_act_split(bool bf16, const Geom& g, int c_alloc, const float* x, void* hi, void* lo,
                     int* counters, int n_counters, cudaStream_t st, int fold) {
    if (g.N == 0) return CB_OK;
    if (fold) {
        if ((reinterpret_cast<uintptr_t>(hi) | reinterpret_cast<uintptr_t>(lo)) & 15)
            return fail(CB_ERR_MISALIGNED, "activation workspace must be 16-byte aligned");
        const int64_t runs = (int64_t)g.N * g.H * g.Q * (c_alloc / (bf16 ? 8 : 4));
        const int blocks = (int)std::min<int64_t>(std::max<int64_t>(1, (runs + 255) / 256),
                                                  (int64_t)sm_count() * 16);
        if (bf16)
            launch_pdl(act_fold_split_kernel<true>, dim3(blocks), 256, 0, st, g, c_alloc, x, hi, lo,
                       counters, n_counters);
        else
            launch_pdl(act_fold_split_kernel<false>, dim3(blocks), 256, 0, st, g, c_alloc, x, hi, lo,
                       counters, n_counters);
        return check_launch("act_fold_split");
    }
    const int64_t in_pix = (int64_t)g.N * g.HW;  // input pixels (not the conv's output npix)
    if (bf16 && g.HW % 4 == 0 && c_alloc % 64 == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0 &&
        !env("CB_K0_NARROW") && (in_pix + AS_PX - 1) / AS_PX <= 0x7fffffffLL) {
        if ((reinterpret_cast<uintptr_t>(hi) | reinterpret_cast<uintptr_t>(lo)) & 15)
            return fail(CB_ERR_MISALIGNED, "activation workspace must be 16-byte aligned");
        const dim3 wgrid((unsigned)((in_pix + AS_PX - 1) / AS_PX), (unsigned)(c_alloc / 64));
        launch_pdl(act_split_wide_kernel, wgrid, 256, 0, st, g.C, g.HW, in_pix, c_alloc, x, hi, lo,
                   counters, n_counters);
        return check_launch("act_split_wide");
    }
    dim3 grid((unsigned)((g.HW + 31) / 32), (unsigned)((c_alloc + 63) / 64), (unsigned)g.N);
    if (grid.z > 65535) return fail(CB_ERR_UNSUPPORTED, "batch too large for act_split grid");
    if ((reinterpret_cast<uintptr_t>(hi) | reinterpret_cast<uintptr_t>(lo)) & 15)
        return fail(CB_ERR_MISALIGNED, "activation workspace must be 16-byte aligned");
    if (bf16)
        launch_pdl(act_split_nhwc_kernel<true>, grid, 256, 0, st, g.C, g.HW, c_alloc, x, hi, lo,
                   counters, n_counters);
    else
        launch_pdl(act_split_nhwc_kernel<false>, grid, 256, 0, st, g.C, g.HW, c_alloc, x, hi, lo,
                   counters, n_counters);
    return check_launch("act_split_nhwc");
}

int launch_weight_split_taps(bool bf16, const Geom& g, int CB, int chk, int kw_pad, const float* w,
                             void* hi, void* lo, cudaStream_t st, int fold, int stack_rs,
                             int k_orig) {
    if (fold && (g.G != 1 || g.S != 1 || chk * CB > WS_CH))
        return fail(CB_ERR_INVALID, "folded weight pack needs one chunk of an R x 1 kernel");
    if ((int64_t)g.K * kw_pad == 0) return CB_OK;
    if ((reinterpret_cast<uintptr_t>(hi) | reinterpret_cast<uintptr_t>(lo)) & 15)
        return fail(CB_ERR_MISALIGNED, "packed weights must be 16-byte aligned");
    if (g.K > 65535) return fail(CB_ERR_UNSUPPORTED, "too many output channels for weight pack");
    const int per_tap = chk * CB;  // multiple of the 16-byte vector (CB >= 16 B / eb)
    const size_t smem = (size_t)WS_CH * g.RS * sizeof(float);
    if (smem > 227 * 1024) return fail(CB_ERR_UNSUPPORTED, "kernel too large for weight pack");
    dim3 grid((unsigned)((per_tap + WS_CH - 1) / WS_CH), (unsigned)g.K);
    auto kern = bf16 ? weight_split_taps_kernel<true> : weight_split_taps_kernel<false>;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return fail(CB_ERR_CUDA, cudaGetErrorString(e));
    }
    kern<<<grid, 256, smem, st>>>(g.K, g.cpg, g.R, g.S, CB, chk, kw_pad, w, hi, lo, fold, stack_rs,
                                  k_orig);
    return check_launch("weight_split_taps");
}

int pre_init_output(const Geom& g, const PixMap& pm, int zero_kind, const float* bias, float* out,
                    cudaStream_t st) {
    if (zero_kind == 1) return launch_fill_bias(g.N, g.K, g.PQ, bias, out, st);
    if (zero_kind == 2) {
        cudaError_t e = cudaMemsetAsync(out, 0, sizeof(float) * (size_t)g.K * pm.j_count, st);
        if (e != cudaSuccess) return fail(CB_ERR_CUDA, cudaGetErrorString(e));
        return CB_OK;
    }
    return fail(CB_ERR_INVALID, "output cannot be pre-initialised for split-K");
}

}  // namespace cb

namespace cb {

// K9 (stacked taps): y[n][f][oy][ox] = bias[f] + sum over the stacked taps of the shifted
// planes of Y', in a fixed tap order (deterministic).  mode 1 (all taps, Y' over the input
// grid): iy = oy*sh - ph + r*dh, ix = ox*sw - pw + s*dw; mode 2 (horizontal taps, Y' over
// output rows x input columns): row oy, ix as above.  Taps outside the image contribute 0.
// One thread per output, consecutive threads along ox.
__global__ void __launch_bounds__(256)
tap_sum_kernel(Geom g, int mode, const float* __restrict__ yp, const float* __restrict__ bias,
               float* __restrict__ y) {
    const int64_t total = (int64_t)g.N * g.K * g.PQ;
    const int T = mode == 1 ? g.RS : g.S;
    const int rows = mode == 1 ? g.H : g.P;
    const int64_t plane = (int64_t)rows * g.W;
    for (int64_t i = blockIdx.x * 256LL + threadIdx.x; i < total; i += (int64_t)gridDim.x * 256) {
        const int64_t nf = i / g.PQ;
        const int pq = (int)(i - nf * g.PQ);
        const int64_t n = nf / g.K;
        const int f = (int)(nf - n * g.K);
        const int oy = pq / g.Q, ox = pq - (pq / g.Q) * g.Q;
        float acc = bias ? __ldg(bias + f) : 0.f;
        const float* base = yp + (n * T * g.K + f) * plane;
        const int nr = mode == 1 ? g.R : 1;
        for (int r = 0; r < nr; ++r) {
            const int iy = mode == 1 ? oy * g.sh - g.ph + r * g.dh : oy;
            if ((unsigned)iy >= (unsigned)rows) continue;
            for (int s = 0; s < g.S; ++s) {
                const int ix = ox * g.sw - g.pw + s * g.dw;
                const int t = mode == 1 ? r * g.S + s : s;
                if ((unsigned)ix < (unsigned)g.W)
                    acc += __ldg(base + (int64_t)t * g.K * plane + (int64_t)iy * g.W + ix);
            }
        }
        y[i] = acc;
    }
}

int launch_tap_sum(const Geom& g, int mode, const float* yp, const float* bias, float* y,
                   cudaStream_t st) {
    const int64_t total = (int64_t)g.N * g.K * g.PQ;
    if (total == 0) return CB_OK;
    const int blocks = (int)std::min<int64_t>((total + 255) / 256, (int64_t)sm_count() * 32);
    tap_sum_kernel<<<blocks, 256, 0, st>>>(g, mode, yp, bias, y);
    return check_launch("tap_sum");
}

}  // namespace cb
