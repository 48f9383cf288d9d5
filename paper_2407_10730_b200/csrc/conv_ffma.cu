// conv_ffma.cu -- SIMT fp32 (FFMA) implicit-GEMM convolution / GEMM: K7 and the FFMA K4.
//
// Same pixel/out-channel/reduction mapping and addressing modes as conv_tc.cu, computed
// with plain fp32 fused multiply-adds (the numerics of a straightforward fp32 conv).  It
// is the variant for shapes where the tensor cores do not pay (tiny C*R*S or K, or
// launch-latency-bound ops), and the independent numerical cross-check of the TC path.
//
// Tile: 128 pixels x 64 output channels x 16 k, 256 threads, 8x4 register blocking,
// register-prefetched double buffering of the next k tile.
#include "cb_common.cuh"

namespace cb {

constexpr int FF_BM = 128, FF_BN = 64, FF_BK = 16, FF_THREADS = 256;

struct FfParams {
    Geom g;
    PixMap pm;
    const float* src;
    const float* w;     // rows x kdim (OIHW flattened), raw fp32
    const float* bias;
    float* out;
    int num_kt;         // k tiles of FF_BK
    int kt_per_split;
    int n_tiles;
    int add_mode;
};

__global__ void __launch_bounds__(FF_THREADS)
conv_ffma_kernel(const __grid_constant__ FfParams p) {
    __shared__ __align__(16) float As[2][FF_BK][FF_BM];
    __shared__ __align__(16) float Bs[2][FF_BK][FF_BN];
    const Geom& g = p.g;
    const int t = threadIdx.x;
    const int tile_m = blockIdx.x;
    const int gi = blockIdx.y / p.n_tiles;
    const int tile_n = blockIdx.y - gi * p.n_tiles;
    const int kt0 = blockIdx.z * p.kt_per_split;
    const int kt1 = min(p.num_kt, kt0 + p.kt_per_split);

    // ---- A loader geometry: pixel row pr, 8 consecutive k at ksub ----
    const int pr = t & (FF_BM - 1);
    const int ksub = (t >> 7) * 8;
    const int64_t jl = (int64_t)tile_m * FF_BM + pr;
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
    const int64_t lrow0 = p.pm.src_mode == SRC_MATRIX ? (int64_t)gi * g.kdim : 0;

    // ---- B loader geometry: out channel bf, 4 consecutive k at bk ----
    const int bf = t >> 2;
    const int bk = (t & 3) * 4;
    const int fl_load = tile_n * FF_BN + bf;
    const bool fvalid = fl_load < g.kpg;
    const float* wrow = p.w + (int64_t)(gi * g.kpg + (fvalid ? fl_load : 0)) * g.kdim;

    float ra[8], rb[4];
    auto load_tile = [&](int kt) {
        const int k0 = kt * FF_BK + ksub;
        if (p.pm.src_mode == SRC_CONV) {
            int c = k0 / g.RS;
            int rs = k0 - c * g.RS;
            int r = rs / g.S;
            int s = rs - r * g.S;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int iy = iy0 + r * g.dh;
                const int ix = ix0 + s * g.dw;
                const bool ok = jvalid && (k0 + i < g.kdim) && (unsigned)iy < (unsigned)g.H &&
                                (unsigned)ix < (unsigned)g.W;
                ra[i] = ok ? __ldg(xb + (int64_t)c * g.HW + iy * g.W + ix) : 0.f;
                if (++s == g.S) {
                    s = 0;
                    if (++r == g.R) {
                        r = 0;
                        ++c;
                    }
                }
            }
        } else {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const bool ok = jvalid && (k0 + i < g.kdim);
                ra[i] = ok ? __ldg(p.src + lbase + (lrow0 + k0 + i) * lstride) : 0.f;
            }
        }
        const int kb0 = kt * FF_BK + bk;
#pragma unroll
        for (int i = 0; i < 4; ++i)
            rb[i] = (fvalid && kb0 + i < g.kdim) ? __ldg(wrow + kb0 + i) : 0.f;
    };
    auto store_tile = [&](int buf) {
#pragma unroll
        for (int i = 0; i < 8; ++i) As[buf][ksub + i][pr] = ra[i];
#pragma unroll
        for (int i = 0; i < 4; ++i) Bs[buf][bk + i][bf] = rb[i];
    };

    const int tm = t & 15, tn = t >> 4;
    float acc[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[i][q] = 0.f;

    if (kt0 < kt1) {
        load_tile(kt0);
        store_tile(0);
        __syncthreads();
        int buf = 0;
        for (int kt = kt0; kt < kt1; ++kt) {
            if (kt + 1 < kt1) load_tile(kt + 1);
#pragma unroll
            for (int kk = 0; kk < FF_BK; ++kk) {
                const float4 a0 = *reinterpret_cast<const float4*>(&As[buf][kk][tm * 4]);
                const float4 a1 = *reinterpret_cast<const float4*>(&As[buf][kk][64 + tm * 4]);
                const float4 b = *reinterpret_cast<const float4*>(&Bs[buf][kk][tn * 4]);
                const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
                const float bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
                for (int i = 0; i < 8; ++i)
#pragma unroll
                    for (int q = 0; q < 4; ++q) acc[i][q] = fmaf(av[i], bv[q], acc[i][q]);
            }
            if (kt + 1 < kt1) {
                store_tile(buf ^ 1);
                __syncthreads();
                buf ^= 1;
            }
        }
    }

    // ---- epilogue ----
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int prow = (i < 4) ? (tm * 4 + i) : (64 + tm * 4 + (i - 4));
        const int64_t jlo = (int64_t)tile_m * FF_BM + prow;
        if (jlo >= p.pm.j_count) continue;
        const int64_t jo = p.pm.j_begin + jlo;
        int64_t obase, ostride;
        dst_linear(g, p.pm, jo, obase, ostride);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int fl = tile_n * FF_BN + tn * 4 + q;
            if (fl >= g.kpg) continue;
            const int f = gi * g.kpg + fl;
            float* dst = p.out + obase + (int64_t)f * ostride;
            if (p.add_mode)
                atomicAdd(dst, acc[i][q]);
            else
                *dst = acc[i][q] + (p.bias ? __ldg(p.bias + f) : 0.f);
        }
    }
}

static int ffma_splits(const Geom& g, int64_t npix, bool allow_split, int num_kt, int n_tiles) {
    const int64_t m_tiles = ceil_div64(npix, FF_BM);
    const int64_t tiles = m_tiles * n_tiles * g.G;
    int splits = 1;
    const int sms = sm_count();
    if (allow_split && tiles < 2 * sms && num_kt >= 8) {
        splits = (int)std::min<int64_t>((2 * sms + tiles - 1) / tiles, num_kt / 4);
        splits = std::max(1, splits);
    }
    const int per = (num_kt + splits - 1) / splits;
    return (num_kt + per - 1) / per;
}

int ffma_plan_query(const Geom& g, int64_t npix, bool allow_split, cb_tile_plan* out) {
    const int num_kt = (g.kdim + FF_BK - 1) / FF_BK;
    const int n_tiles = (g.kpg + FF_BN - 1) / FF_BN;
    out->variant = CB_VARIANT_FFMA;
    out->block_m = FF_BM;
    out->block_n = FF_BN;
    out->block_k = FF_BK;
    out->stages = 2;
    out->splits = ffma_splits(g, npix, allow_split, num_kt, n_tiles);
    out->m_tiles = ceil_div64(npix, FF_BM);
    out->n_tiles = (int64_t)n_tiles * g.G;
    out->k_blocks = num_kt;
    out->ctas = out->m_tiles * out->n_tiles * out->splits;
    return CB_OK;
}

int pre_init_output(const Geom& g, const PixMap& pm, int zero_kind, const float* bias, float* out,
                    cudaStream_t st);

int launch_ffma(const Geom& g, const PixMap& pm, const float* src, const float* w,
                const float* bias, float* out, int add_mode, int zero_kind, cudaStream_t st) {
    if (pm.j_count == 0) return CB_OK;
    FfParams prm{};
    prm.g = g;
    prm.pm = pm;
    prm.src = src;
    prm.w = w;
    prm.bias = bias;
    prm.out = out;
    prm.num_kt = (g.kdim + FF_BK - 1) / FF_BK;
    prm.n_tiles = (g.kpg + FF_BN - 1) / FF_BN;
    prm.add_mode = add_mode;
    const int64_t m_tiles = ceil_div64(pm.j_count, FF_BM);
    int splits = ffma_splits(g, pm.j_count, add_mode || zero_kind != 0, prm.num_kt, prm.n_tiles);
    prm.kt_per_split = (prm.num_kt + splits - 1) / splits;
    splits = (prm.num_kt + prm.kt_per_split - 1) / prm.kt_per_split;
    if (splits > 1 && !add_mode) {
        int rc = pre_init_output(g, pm, zero_kind, bias, out, st);
        if (rc) return rc;
        prm.add_mode = 1;
    }
    if (m_tiles > 0x7fffffffLL) return fail(CB_ERR_UNSUPPORTED, "too many pixel tiles");
    dim3 grid((unsigned)m_tiles, (unsigned)(prm.n_tiles * g.G), (unsigned)splits);
    conv_ffma_kernel<<<grid, FF_THREADS, 0, st>>>(prm);
    return check_launch("conv_ffma_kernel");
}

}  // namespace cb
