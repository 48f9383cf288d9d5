"""GPU parity: every kernel of the path against the CPU oracle on identical seeded inputs.

Gate (BASELINE.json north_star): max|y - y_ref| / sqrt(C/g*R*S) <= 1e-4 for
convolutions (written below as TOL); packing kernels are bit-exact.
"""

from __future__ import annotations

import numpy as np
import pytest

from corpus import cfg, corpus
from oracle import conv_oracle as orc

pytestmark = pytest.mark.gpu

TOL = 1e-4
VARIANTS = ["tc3xtf32", "tc3xbf16", "ffma"]


def _inputs(d, seed=0):
    from paper_2407_10730_b200.algos import ConvInputs
    x, w, b = orc.make_inputs(d, seed)
    return ConvInputs(desc=d, input=x, weights=w, bias=b), (x, w, b)


def _check_conv(d, got, ref, tol=TOL):
    assert got.shape == ref.shape and got.dtype == np.float32
    err = orc.normalized_max_err(got, ref, orc.reduction_len(d))
    assert err <= tol, f"{d}: normalized max err {err:.3e} > {tol:g}"
    return err


SMALL = corpus(24, seed=7, spatial=(9, 14)) + corpus(6, seed=8, spatial=(5, 9), batch=(2, 3))
SUPPORTED = corpus(12, seed=31, spatial=(8, 14), supported_only=True) + \
    corpus(4, seed=32, spatial=(6, 10), supported_only=True, batch=(2, 3))


@pytest.mark.parametrize("variant", VARIANTS)
def test_fused_matches_oracle_on_corpus(cuda, variant):
    from paper_2407_10730_b200.algos import conv_fused
    for d in SMALL:
        inp, (x, w, b) = _inputs(d)
        _check_conv(d, conv_fused(inp, variant=variant), orc.conv_direct_naive(d, x, w, b))


@pytest.mark.parametrize("cg,bn", [(1, 64), (1, 128), (1, 256), (2, 128), (2, 256)])
@pytest.mark.parametrize("variant", ["tc3xtf32", "tc3xbf16"])
def test_fused_every_tile_config(cuda, variant, cg, bn, monkeypatch):
    """Force each TMA tile configuration (1-CTA / CTA pair x BN) on ragged shapes:
    partial pixel tiles, partial channel tiles, batch > 1, stride, padding, groups."""
    from paper_2407_10730_b200.algos import conv_fused, fused_layout
    from paper_2407_10730_b200.descriptor import ConvDescriptor
    monkeypatch.setenv("CB_TMA_CG", str(cg))
    monkeypatch.setenv("CB_TMA_BN", str(bn))
    shapes = SMALL[:10] + [
        ConvDescriptor(batch=3, in_channels=64, in_h=15, in_w=13, out_channels=200, k_h=3, k_w=3,
                       pad_h=1, pad_w=1, has_bias=True),
        ConvDescriptor(batch=2, in_channels=96, in_h=17, in_w=17, out_channels=72, k_h=3, k_w=3,
                       stride_h=2, stride_w=2, pad_h=1, pad_w=1),
        ConvDescriptor(batch=5, in_channels=32, in_h=9, in_w=9, out_channels=256, k_h=1, k_w=1),
        ConvDescriptor(batch=2, in_channels=64, in_h=12, in_w=12, out_channels=64, k_h=3, k_w=3,
                       pad_h=1, pad_w=1, groups=2),
    ]
    n_tma = 0
    for d in shapes:
        inp, (x, w, b) = _inputs(d)
        n_tma += fused_layout(d, variant)["path"]
        _check_conv(d, conv_fused(inp, variant=variant), orc.conv_direct_naive(d, x, w, b))
    assert n_tma >= 4


@pytest.mark.parametrize("cg", [1, 2])
def test_fused_tail_split(cuda, cg, monkeypatch):
    """Grids with more tiles than clusters and a ragged last wave: the tail tiles are
    split along K and reduced by the last-arriving part (deterministic fixup)."""
    from paper_2407_10730_b200.algos import conv_fused, fused_plan
    from paper_2407_10730_b200.descriptor import ConvDescriptor
    monkeypatch.setenv("CB_TMA_CG", str(cg))
    # PQ % 4 == 0 (vector fixup stores through a smem transpose) and PQ odd (direct stores)
    for hw in (16, 15):
        monkeypatch.delenv("CB_TMA_TAIL", raising=False)
        monkeypatch.delenv("CB_TMA_TAIL_LAST", raising=False)
        d = ConvDescriptor(batch=80, in_channels=64, in_h=hw, in_w=hw, out_channels=64, k_h=3,
                           k_w=3, pad_h=1, pad_w=1, has_bias=True)
        assert fused_plan(d)["m_tiles"] > 0
        inp, (x, w, b) = _inputs(d)
        ref = orc.conv_im2col64(d, x, w, b)
        y1 = conv_fused(inp)
        y2 = conv_fused(inp)
        _check_conv(d, y1, ref)
        assert np.array_equal(y1, y2), "tail fixup must be deterministic"
        # tail parts last (the old item order): the same sums in the same order, same bits
        monkeypatch.setenv("CB_TMA_TAIL_LAST", "1")
        assert np.array_equal(conv_fused(inp), y1)
        monkeypatch.setenv("CB_TMA_TAIL", "0")
        _check_conv(d, conv_fused(inp), ref)


@pytest.mark.parametrize("variant", VARIANTS)
def test_im2col_gemm_matches_oracle_on_corpus(cuda, variant):
    from paper_2407_10730_b200.algos import conv_baseline_im2col_gemm
    from paper_2407_10730_b200.timing import PhaseLedger
    for d in SMALL:
        inp, (x, w, b) = _inputs(d)
        got = conv_baseline_im2col_gemm(inp, PhaseLedger(), variant=variant)
        _check_conv(d, got, orc.conv_direct_naive(d, x, w, b))


@pytest.mark.parametrize("variant", VARIANTS)
def test_sconv_matches_oracle_on_supported(cuda, variant):
    from paper_2407_10730_b200.algos import CacheParams, conv_main_blocked_direct
    from paper_2407_10730_b200.timing import PhaseLedger
    for i, d in enumerate(SUPPORTED):
        inp, (x, w, b) = _inputs(d)
        # alternate default plan and a tiny budget that forces many slices / chunks
        cache = None if i % 2 == 0 else CacheParams(l2_bytes=8 * 1024)
        got = conv_main_blocked_direct(inp, PhaseLedger(), cache=cache, variant=variant)
        _check_conv(d, got, orc.conv_direct_naive(d, x, w, b))


def test_im2col_bit_exact(cuda):
    from paper_2407_10730_b200.algos import im2col_transform
    for d in SMALL + [cfg("cfg1"), cfg("cfg2a"), cfg("cfg2b"), cfg("cfg3"), cfg("cfg4")]:
        inp, (x, _, _) = _inputs(d)
        got = im2col_transform(inp)
        want = orc.im2col(d, x)
        assert got.shape == want.shape
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), d


def test_slice_pack_bit_exact(cuda):
    import torch
    from paper_2407_10730_b200 import _capi
    import ctypes
    lib = _capi.load()
    for d in SUPPORTED[:8] + [cfg("cfg3", batch=2)]:
        _, (x, _, _) = _inputs(d)
        oh, ow = orc.output_shape(d)
        for band in (1, 3, oh):
            cd = _capi.cdesc(d)
            sp = _capi.CbSlicePlan()
            _capi.check(lib.cb_sconv_plan(ctypes.byref(cd), band * ow, ctypes.byref(sp)))
            assert sp.band_rows == min(band, oh)
            first, count = sp.num_slices // 3, max(1, sp.num_slices - sp.num_slices // 3 - 1)
            want = orc.slice_pack(d, x, sp.band_rows, first, count)
            xd = torch.from_numpy(x).cuda()
            out = torch.full((want.size + 64,), float("nan"), device="cuda")
            _capi.check(lib.cb_sconv_pack_f32(ctypes.byref(cd), ctypes.byref(sp), first, count,
                                              xd.data_ptr(), out.data_ptr(),
                                              torch.cuda.current_stream().cuda_stream))
            got = out.cpu().numpy()
            assert np.array_equal(got[:want.size].view(np.uint32), want.view(np.uint32)), (d, band)
            assert np.isnan(got[want.size:]).all(), "pack wrote past its slice range"


@pytest.mark.parametrize("variant", VARIANTS)
def test_gemm_dropin(cuda, variant):
    from paper_2407_10730_b200.algos import GemmBlocking, gemm
    from paper_2407_10730_b200.timing import PhaseLedger
    rng = np.random.default_rng(1)
    for m, k, n in [(17, 13, 19), (1, 1, 1), (64, 300, 257), (300, 77, 1000)]:
        a = (rng.random((m, k), dtype=np.float32) * 2 - 1)
        b = (rng.random((k, n), dtype=np.float32) * 2 - 1)
        c = (rng.random((m, n), dtype=np.float32) * 2 - 1)
        want = a.astype(np.float64) @ b.astype(np.float64) + c
        gemm(a, b, c, GemmBlocking(), PhaseLedger(), variant=variant)
        err = float(np.abs(c - want).max()) / np.sqrt(k)
        assert err <= TOL, (m, k, n, err)
    # reference known answers (test_algos.py:95-125)
    a = np.array([[3.0]], np.float32)
    c = np.zeros((1, 1), np.float32)
    gemm(a, np.array([[-2.0]], np.float32), c, GemmBlocking(), PhaseLedger(), variant=variant)
    assert c[0, 0] == -6.0
    c = np.full((2, 2), 10.0, np.float32)
    gemm(np.ones((2, 2), np.float32), np.ones((2, 2), np.float32), c, GemmBlocking(),
         PhaseLedger(), variant=variant)
    assert (c == 12.0).all()


@pytest.mark.parametrize("name", ["cfg1", "cfg2a", "cfg2b", "cfg3", "cfg4"])
def test_baseline_configs_all_paths(cuda, name):
    """The five BASELINE.json configurations at full size through all three algorithms."""
    from paper_2407_10730_b200.algos import (conv_baseline_im2col_gemm, conv_fused,
                                             conv_main_blocked_direct)
    from paper_2407_10730_b200.timing import PhaseLedger
    d = cfg(name)
    inp, (x, w, b) = _inputs(d)
    ref = orc.conv_im2col64(d, x, w, b)
    errs = {}
    for variant in ("tc3xtf32", "tc3xbf16"):
        errs[("fused", variant)] = _check_conv(d, conv_fused(inp, variant=variant), ref)
    errs[("fused", "ffma")] = _check_conv(d, conv_fused(inp, variant="ffma"), ref)
    errs["im2col"] = _check_conv(d, conv_baseline_im2col_gemm(inp, PhaseLedger()), ref)
    errs["sconv"] = _check_conv(d, conv_main_blocked_direct(inp, PhaseLedger()), ref)
    print(name, {str(k): f"{v:.2e}" for k, v in errs.items()})


def test_known_answers(cuda):
    """All-ones 3x3 with bias 0.5 -> 9.5 everywhere (reference test_algos.py:193-200)."""
    from paper_2407_10730_b200.algos import (ConvInputs, conv_baseline_im2col_gemm, conv_fused,
                                             conv_main_blocked_direct)
    from paper_2407_10730_b200.descriptor import ConvDescriptor
    from paper_2407_10730_b200.timing import PhaseLedger
    d = ConvDescriptor(batch=1, in_channels=1, in_h=5, in_w=5, out_channels=1, k_h=3, k_w=3,
                       has_bias=True)
    inp = ConvInputs(desc=d, input=np.ones((1, 1, 5, 5), np.float32),
                     weights=np.ones((1, 1, 3, 3), np.float32), bias=np.full(1, 0.5, np.float32))
    for fn in (conv_baseline_im2col_gemm, conv_main_blocked_direct):
        assert (fn(inp, PhaseLedger()) == 9.5).all()
    for v in VARIANTS:
        assert (conv_fused(inp, variant=v) == 9.5).all()


@pytest.mark.parametrize("name", ["cfg1", "cfg2a"])
def test_host_pipeline_matches_dropin(cuda, name):
    """HostPipeline (streamed host buffers) gives the drop-in's bits, step after step, and
    matches the oracle."""
    import torch
    from paper_2407_10730_b200.algos import HostPipeline, conv_fused
    d = cfg(name)
    inp, (x, w, b) = _inputs(d)
    v = "tc3xbf16"  # bitwise comparison: a deterministic variant (ffma split-K uses atomics)
    want = conv_fused(inp, variant=v)
    pipe = HostPipeline(d, variant=v)
    xs = [torch.from_numpy(x).pin_memory(), torch.from_numpy(x[:, ::-1].copy()).pin_memory()]
    wp = torch.from_numpy(w).pin_memory()
    ys = [torch.empty(want.shape, dtype=torch.float32).pin_memory() for _ in range(3)]
    for i in range(3):  # more steps than buffer slots: slot reuse is ordered by events
        pipe.submit(xs[i % 2], wp, ys[i])
    pipe.synchronize()
    assert np.array_equal(ys[0].numpy(), want) and np.array_equal(ys[2].numpy(), want)
    flipped = conv_fused(_inputs(d)[0].__class__(desc=d, input=x[:, ::-1].copy(), weights=w),
                         variant=v)
    assert np.array_equal(ys[1].numpy(), flipped)
    _check_conv(d, ys[0].numpy(), orc.conv_direct_naive(d, x, w, b))


@pytest.mark.parametrize("mode", ["fused", "baseline", "main"])
def test_run_single_graph_mode(cuda, mode):
    """Graph-replayed timing reports the same phases and call counts as eager timing."""
    from paper_2407_10730_b200.harness import RunConfig, run_single
    d = cfg("cfg1")
    eager = run_single(d, RunConfig(mode=mode, warmups=1, runs=2))
    graph = run_single(d, RunConfig(mode=mode, warmups=1, runs=3, graph=True))
    assert eager.status == graph.status == "ok", (eager.detail, graph.detail)
    assert dict(graph.stats.calls) == dict(eager.stats.calls)
    assert graph.stats.operation_ns_mean > 0


STACKED = [  # few output channels, many input channels: the stacked-tap path (fused path 3)
    dict(batch=2, in_channels=128, in_h=17, in_w=23, out_channels=8, k_h=3, k_w=3, stride_h=1,
         stride_w=1, pad_h=1, pad_w=1, has_bias=True),
    dict(batch=1, in_channels=256, in_h=20, in_w=20, out_channels=16, k_h=3, k_w=3, stride_h=2,
         stride_w=2, pad_h=1, pad_w=1),
    dict(batch=1, in_channels=192, in_h=15, in_w=16, out_channels=4, k_h=5, k_w=5, stride_h=1,
         stride_w=1, pad_h=2, pad_w=2, dil_h=2, dil_w=2, has_bias=True),
    dict(batch=3, in_channels=160, in_h=9, in_w=11, out_channels=10, k_h=1, k_w=7, stride_h=1,
         stride_w=2, pad_h=0, pad_w=3),
    # row stacking (S*K <= 256 < R*S*K): only the horizontal taps are stacked
    dict(batch=1, in_channels=64, in_h=19, in_w=21, out_channels=32, k_h=7, k_w=7, stride_h=1,
         stride_w=1, pad_h=3, pad_w=3, has_bias=True),
    dict(batch=2, in_channels=96, in_h=16, in_w=18, out_channels=24, k_h=5, k_w=5, stride_h=2,
         stride_w=2, pad_h=2, pad_w=1, dil_h=1, dil_w=2),
]


@pytest.mark.parametrize("variant", ["tc3xbf16", "tc3xtf32"])
@pytest.mark.parametrize("spec", range(len(STACKED)))
def test_stacked_taps_match_oracle(cuda, variant, spec):
    from paper_2407_10730_b200.algos import conv_fused, fused_layout
    from paper_2407_10730_b200.descriptor import ConvDescriptor
    d = ConvDescriptor(**STACKED[spec])
    assert fused_layout(d, variant)["path"] == 1  # TMA kernel on the stacked 1x1 geometry
    inp, (x, w, b) = _inputs(d)
    _check_conv(d, conv_fused(inp, variant=variant), orc.conv_direct_naive(d, x, w, b))


@pytest.mark.parametrize("variant", ["tc3xtf32", "tc3xbf16"])
def test_stepwise_gemm_odd_chunk_counts(cuda, variant):
    """K8 with an odd number of 32-wide reduction chunks per item and several items per CTA
    (the chunk-to-producer-group assignment must stay fixed across items), back to back."""
    from paper_2407_10730_b200.algos import conv_baseline_im2col_gemm, conv_main_blocked_direct
    from paper_2407_10730_b200.descriptor import ConvDescriptor
    from paper_2407_10730_b200.timing import PhaseLedger
    shapes = [ConvDescriptor(batch=1, in_channels=32, in_h=28, in_w=28, out_channels=32, k_h=1,
                             k_w=1, stride_h=2, stride_w=2),                       # 1 chunk
              ConvDescriptor(batch=1, in_channels=32, in_h=164, in_w=164, out_channels=32, k_h=3,
                             k_w=3, pad_h=1, pad_w=1)]                             # 9 chunks, 211 tiles
    for _ in range(2):
        for d in shapes:
            inp, (x, w, b) = _inputs(d)
            ref = orc.conv_direct_naive(d, x, w, b)
            for fn in (conv_baseline_im2col_gemm, conv_main_blocked_direct):
                _check_conv(d, fn(inp, PhaseLedger(), variant=variant), ref)


def _model_ops(max_flops: float, step: int):
    import json
    from pathlib import Path
    from paper_2407_10730_b200.descriptor import flop_count, parse_key
    data = json.loads((Path(__file__).resolve().parent.parent / "configs" / "model_ops.json").read_text())
    ds = [parse_key(k) for k in data["unique"]]
    return [d for d in ds if flop_count(d) <= max_flops][::step]


@pytest.mark.parametrize("variant", ["tc3xbf16", "auto"])
def test_model_layers_match_oracle(cuda, variant):
    """Real-network layers (torchvision, configs/model_ops.json) that are cheap to check:
    depthwise / grouped / dilated / 1x1 / strided shapes through the fused path and
    Im2col-GEMM."""
    from paper_2407_10730_b200.algos import conv_baseline_im2col_gemm, conv_fused
    from paper_2407_10730_b200.timing import PhaseLedger
    ops = _model_ops(2e7, 4)
    assert len(ops) >= 20
    for d in ops:
        inp, (x, w, b) = _inputs(d)
        ref = orc.conv_direct_naive(d, x, w, b)
        _check_conv(d, conv_fused(inp, variant=variant), ref)
        if variant == "auto":
            _check_conv(d, conv_baseline_im2col_gemm(inp, PhaseLedger()), ref)


# K7 (path 2): every compile-time producer layout (conv_ts.cu CB_TS_FIXED_LIST) and the
# generic offset-table producer, unit and even horizontal stride (the bank-swap lanes),
# odd output sizes (a partial last tile), bias, batch > 1, dilation (generic only).
K7_SHAPES = [(3, 7, 7), (3, 3, 3), (3, 5, 5), (4, 3, 3), (4, 7, 7), (2, 5, 3), (8, 3, 3)]


@pytest.mark.parametrize("crs", K7_SHAPES)
@pytest.mark.parametrize("stride", [1, 2])
@pytest.mark.parametrize("generic", [False, True, "no_pair", "padded_pairs"])
def test_direct_few_channel_conv(cuda, crs, stride, generic, monkeypatch):
    from paper_2407_10730_b200.algos import conv_fused, fused_layout
    from paper_2407_10730_b200.descriptor import ConvDescriptor
    c, r, s = crs
    if generic == "no_pair":  # compile-time producers in plain OIHW order (one LDS per tap)
        monkeypatch.setenv("CB_TS_NO_PAIR", "1")
        generic = False
    elif generic == "padded_pairs":  # one zero pad tap per row instead of the mixed layout
        monkeypatch.setenv("CB_TS_PAIRMODE", "1")
        generic = False
    elif generic:
        monkeypatch.setenv("CB_TS_GENERIC", "1")
    for d in (ConvDescriptor(batch=2, in_channels=c, in_h=37, in_w=44, out_channels=24, k_h=r, k_w=s,
                             stride_h=stride, stride_w=stride, pad_h=r // 2, pad_w=s // 2, has_bias=True),
              ConvDescriptor(batch=1, in_channels=c, in_h=20, in_w=28,
                             out_channels=64 if c * r * s <= 160 else 32, k_h=r, k_w=s,
                             stride_h=2, stride_w=stride, pad_h=r // 2, pad_w=s // 2, dil_h=2,
                             dil_w=2 if generic else 1)):
        assert fused_layout(d, "tc3xbf16")["path"] == 2, d
        inp, (x, w, b) = _inputs(d)
        _check_conv(d, conv_fused(inp, variant="tc3xbf16"), orc.conv_direct_naive(d, x, w, b))


@pytest.mark.parametrize("crs", [(3, 7, 7), (3, 3, 3), (3, 5, 5), (4, 3, 3), (4, 7, 7)])
@pytest.mark.parametrize("stride", [1, 2])
@pytest.mark.parametrize("layout", ["default", "plain"])
def test_direct_few_channel_conv_tf32(cuda, crs, stride, layout, monkeypatch):
    """K7 with the 3xTF32 split (tf32 words in TMEM, kind::tf32 MMAs, one or two A buffers):
    every compile-time layout, the mixed and the plain reduction order, odd output sizes,
    bias, batch > 1, many tiles per CTA."""
    from paper_2407_10730_b200.algos import conv_fused, fused_layout
    from paper_2407_10730_b200.descriptor import ConvDescriptor
    c, r, s = crs
    if layout == "plain":
        monkeypatch.setenv("CB_TS_NO_PAIR", "1")
    for d in (ConvDescriptor(batch=2, in_channels=c, in_h=37, in_w=44, out_channels=24, k_h=r, k_w=s,
                             stride_h=stride, stride_w=stride, pad_h=r // 2, pad_w=s // 2, has_bias=True),
              ConvDescriptor(batch=3, in_channels=c, in_h=160, in_w=192,
                             out_channels=64 if c * r * s <= 100 else 32, k_h=r, k_w=s,
                             stride_h=2, stride_w=stride, pad_h=r // 2, pad_w=s // 2)):
        assert fused_layout(d, "tc3xtf32")["path"] == 2, d
        inp, (x, w, b) = _inputs(d)
        _check_conv(d, conv_fused(inp, variant="tc3xtf32"), orc.conv_direct_naive(d, x, w, b))


def test_direct_few_channel_conv_is_repeatable(cuda):
    """K7's pipeline (window ring, TMEM A ring, two accumulators, cross-tile barrier tests)
    gives bit-identical results launch after launch on a grid with many tiles per CTA."""
    import torch
    from paper_2407_10730_b200.algos import conv_fused, fused_layout
    from paper_2407_10730_b200.descriptor import ConvDescriptor
    d = ConvDescriptor(batch=12, in_channels=3, in_h=224, in_w=224, out_channels=64, k_h=7, k_w=7,
                       stride_h=2, stride_w=2, pad_h=3, pad_w=3)
    assert fused_layout(d, "tc3xbf16")["path"] == 2
    g = torch.Generator(device="cuda").manual_seed(3)
    x = torch.rand((d.batch, 3, 224, 224), device="cuda", generator=g) * 2 - 1
    w = torch.rand((64, 3, 7, 7), device="cuda", generator=g) * 2 - 1
    from paper_2407_10730_b200.algos import ConvInputs
    inp = ConvInputs(desc=d, input=x, weights=w)
    first = conv_fused(inp, variant="tc3xbf16").clone()
    for _ in range(40):
        assert torch.equal(conv_fused(inp, variant="tc3xbf16"), first)
    ref = torch.nn.functional.conv2d(x[:2].double().cpu(), w.double().cpu(), stride=2, padding=3)
    err = (first[:2].double().cpu() - ref).abs().max().item() / (3 * 7 * 7) ** 0.5
    assert err <= 1e-4, err


@pytest.mark.parametrize("variant", ["tc3xbf16", "tc3xtf32"])
def test_short_grid_many_k_parts(cuda, variant):
    """Few output tiles with a long reduction: each tile is cut into up to 16 K parts
    (fixup sums the parts in groups of 4, in part order); deterministic and within tolerance."""
    from paper_2407_10730_b200.algos import conv_fused, fused_plan
    from paper_2407_10730_b200.descriptor import ConvDescriptor
    d = ConvDescriptor(batch=1, in_channels=1024, in_h=14, in_w=14, out_channels=64, k_h=3, k_w=3,
                       pad_h=1, pad_w=1, has_bias=True)
    plan = fused_plan(d, variant)
    assert plan["ctas"] > 4 * plan["m_tiles"] * plan["n_tiles"], plan  # more than 4 parts a tile
    inp, (x, w, b) = _inputs(d)
    y1 = conv_fused(inp, variant=variant)
    _check_conv(d, y1, orc.conv_im2col64(d, x, w, b))
    assert np.array_equal(y1, conv_fused(inp, variant=variant))


def test_activation_split_variants_agree(cuda, monkeypatch):
    """K0's wide (flattened pixels, float4 loads, swizzled tile) and narrow variants write the
    same split halves: the fused conv's result is bitwise the same with either."""
    from paper_2407_10730_b200.algos import conv_fused
    from paper_2407_10730_b200.descriptor import ConvDescriptor
    d = ConvDescriptor(batch=3, in_channels=96, in_h=10, in_w=14, out_channels=40, k_h=3, k_w=3,
                       pad_h=1, pad_w=1, has_bias=True)
    inp, (x, w, b) = _inputs(d)
    y_wide = conv_fused(inp, variant="tc3xbf16")
    _check_conv(d, y_wide, orc.conv_direct_naive(d, x, w, b))
    monkeypatch.setenv("CB_K0_NARROW", "1")
    assert np.array_equal(conv_fused(inp, variant="tc3xbf16"), y_wide)


def _sweep_classes(max_flops: float, per_class: int) -> dict:
    """Config-5 sweep ops grouped by the fused path / plan the planner picks for them
    (ffma, gather, K7 direct, stacked taps, folded taps, K parts > 4 per tile, tail split,
    plain TMA tiles): the cheapest `per_class` and the largest `per_class` ops of each class
    under `max_flops`."""
    from paper_2407_10730_b200 import algos, configs
    from paper_2407_10730_b200.descriptor import flop_count
    out: dict = {}
    for d in sorted(set(configs.sweep()), key=lambda d: (flop_count(d), str(d))):
        if flop_count(d) > max_flops:
            continue
        v = algos.resolve_variant(d, "auto")
        if v == "ffma":
            out.setdefault("ffma", []).append(d)
            continue
        lay = algos.fused_layout(d, v)
        if lay["path"] != 1:
            out.setdefault(f"path{lay['path']}", []).append(d)
            continue
        plan = algos.fused_plan(d, v)
        tiles = plan["m_tiles"] * plan["n_tiles"]
        if lay["weight_rows"] != d.out_channels:
            out.setdefault("stacked", []).append(d)
        elif d.k_w > 1 and lay["chunk_channels"] >= d.in_channels * d.k_w:
            out.setdefault("folded", []).append(d)
        key = "parts>4" if plan["ctas"] > 4 * tiles else "split" if plan["ctas"] > tiles else "plain"
        out.setdefault(key, []).append(d)
    picked = {k: v[:per_class] + v[per_class:][-per_class:] for k, v in out.items()}
    # the many-part tail split of the widest reductions (C=2048, 5x5 / 7x7)
    wide = [d for d in out.get("parts>4", []) if d.in_channels == 2048 and d.k_h in (5, 7)]
    picked["parts>4"] += [d for d in wide[::max(1, len(wide) // per_class)] if d not in picked["parts>4"]]
    return picked


def test_sweep_plan_classes_match_oracle(cuda):
    """Config-5 ops from every planner class -- including the many-K-part tail split of
    C=2048 5x5 / 7x7 reductions, tap stacking, tap folding and K7 -- through the fused
    (auto), Im2col-GEMM and SConv paths, against the float64 oracle on make_inputs data.
    (tests/sweep_parity.py runs the same check on all 9243 ops.)"""
    from paper_2407_10730_b200.algos import (conv_baseline_im2col_gemm, conv_fused,
                                             conv_main_blocked_direct)
    from paper_2407_10730_b200.timing import PhaseLedger
    classes = _sweep_classes(3e9, 3)
    for want in ("ffma", "path2", "stacked", "folded", "parts>4", "split", "plain"):
        assert len(classes.get(want, [])) >= 2, (want, sorted(classes))
    assert any(d.in_channels == 2048 and d.k_h in (5, 7) for d in classes["parts>4"])
    worst = {}
    for name, ds in classes.items():
        for d in ds:
            inp, (x, w, b) = _inputs(d)
            ref = orc.conv_banded64(d, x, w, b).astype(np.float32)
            for path, fn in (("fused", lambda: conv_fused(inp)),
                             ("im2col", lambda: conv_baseline_im2col_gemm(inp, PhaseLedger())),
                             ("sconv", lambda: conv_main_blocked_direct(inp, PhaseLedger()))):
                e = _check_conv(d, fn(), ref)
                worst[(name, path)] = max(worst.get((name, path), 0.0), e)
    print({f"{k[0]}/{k[1]}": f"{v:.1e}" for k, v in sorted(worst.items())})


PROMOTE_KEYS = ["n1_c2048x28x28_f256x7x7_s1x1_p3x3_d1x1_g1_b0",     # C*R*S = 100352, few tiles
                "n1_c2048x112x112_f128x3x3_s1x1_p1x1_d1x1_g1_b0",   # 18432, many whole tiles
                "n1_c1024x28x28_f64x7x7_s2x2_p3x3_d1x1_g1_b0"]      # 50176, short grid (K parts)


@pytest.mark.parametrize("key", PROMOTE_KEYS)
def test_large_reductions_with_accumulator_promotion(cuda, key):
    """The tcgen05 fp32 accumulation truncates: one accumulator over C*R*S = 100352 drifted
    to 1.3e-3 (3xTF32) / 6e-4 (3xBF16) normalized error on the config-5 sweep.  Every
    tensor-core path drains its accumulator every ~2-4K reduction elements (promote_k) and
    adds the partials in fp32; all of them must now pass the gate on these reductions."""
    from paper_2407_10730_b200.algos import (conv_baseline_im2col_gemm, conv_fused,
                                             conv_main_blocked_direct)
    from paper_2407_10730_b200.descriptor import parse_key
    from paper_2407_10730_b200.timing import PhaseLedger
    d = parse_key(key)
    inp, (x, w, b) = _inputs(d)
    ref = orc.conv_banded64(d, x, w, b).astype(np.float32)
    errs = {}
    for v in ("tc3xbf16", "tc3xtf32"):
        errs[f"fused/{v}"] = _check_conv(d, conv_fused(inp, variant=v), ref)
        errs[f"im2col/{v}"] = _check_conv(d, conv_baseline_im2col_gemm(inp, PhaseLedger(), variant=v), ref)
        errs[f"sconv/{v}"] = _check_conv(d, conv_main_blocked_direct(inp, PhaseLedger(), variant=v), ref)
    print(key, {k: f"{e:.1e}" for k, e in errs.items()})


# K8's ragged last wave: cfg4-like shapes with more pixel tiles than SMs.  Both tails -- the
# default channel split and the K split (CB_K8_KSPLIT: parts add into y in part order
# through hand-off flags) -- must match the oracle and be bitwise reproducible.
KSPLIT = [dict(batch=32, in_channels=64, in_h=28, in_w=28, out_channels=96, k_h=3, k_w=3,
               pad_h=1, pad_w=1, has_bias=True),
          dict(batch=40, in_channels=32, in_h=20, in_w=20, out_channels=256, k_h=5, k_w=5,
               pad_h=2, pad_w=2, stride_h=1, stride_w=1)]


@pytest.mark.parametrize("spec", range(len(KSPLIT)))
def test_stepwise_tail_splits(cuda, spec, monkeypatch):
    from paper_2407_10730_b200.algos import conv_baseline_im2col_gemm
    from paper_2407_10730_b200.descriptor import ConvDescriptor
    from paper_2407_10730_b200.timing import PhaseLedger
    d = ConvDescriptor(**KSPLIT[spec])
    inp, (x, w, b) = _inputs(d)
    ref = orc.conv_im2col64(d, x, w, b)
    y0 = conv_baseline_im2col_gemm(inp, PhaseLedger())
    _check_conv(d, y0, ref)
    for parts in ("2", "3"):
        monkeypatch.setenv("CB_K8_KSPLIT", parts)
        y1 = conv_baseline_im2col_gemm(inp, PhaseLedger())
        y2 = conv_baseline_im2col_gemm(inp, PhaseLedger())
        _check_conv(d, y1, ref)
        assert np.array_equal(y1.view(np.uint32), y2.view(np.uint32)), "K-split tail not deterministic"



@pytest.mark.parametrize("mode", ["CB_TMA_TSTORE"])
def test_fused_tma_store_modes_bitwise(cuda, mode, monkeypatch):
    """K6's opt-in TMA-store epilogue (128-pixel boxes for tiles inside one image) stores the
    same values as the default per-lane stores: tiles inside and across images, bias, a
    partial channel chunk."""
    from paper_2407_10730_b200.algos import conv_fused
    from paper_2407_10730_b200.descriptor import ConvDescriptor
    for d in (cfg("cfg4", batch=4),
              ConvDescriptor(batch=3, in_channels=64, in_h=15, in_w=12, out_channels=200, k_h=3, k_w=3,
                             pad_h=1, pad_w=1, has_bias=True)):
        inp, (x, w, b) = _inputs(d)
        y0 = conv_fused(inp, variant="tc3xbf16")
        monkeypatch.setenv(mode, "1")
        y1 = conv_fused(inp, variant="tc3xbf16")
        monkeypatch.delenv(mode)
        assert np.array_equal(y0.view(np.uint32), y1.view(np.uint32)), d
