"""The C-ABI library on a host without a GPU: it loads, exports exactly the symbols
include/convb200.h declares, and its host-only entry points (validation, shapes, plans,
workspace sizing) behave like the reference data model.  No kernel launches here."""

from __future__ import annotations

import ctypes
import re
import subprocess
from pathlib import Path

import pytest

from paper_2407_10730_b200 import _capi
from paper_2407_10730_b200.descriptor import ConvDescriptor, InvalidDescriptorError, output_shape

ROOT = Path(__file__).resolve().parent.parent


@pytest.fixture(scope="module")
def lib():
    if not _capi.LIB_PATH.exists():
        from paper_2407_10730_b200.build import build
        build()
    return _capi.load()


def header_symbols() -> set[str]:
    text = (ROOT / "include" / "convb200.h").read_text()
    return set(re.findall(r"^\s*(?:int|int32_t|uint64_t|const char\*)\s+(cb_\w+)\s*\(", text, re.M))


def test_exports_match_header(lib):
    declared = header_symbols()
    assert declared == set(_capi.EXPORTS), declared ^ set(_capi.EXPORTS)
    nm = subprocess.run(["nm", "-D", "--defined-only", str(_capi.LIB_PATH)], capture_output=True,
                        text=True, check=True).stdout
    exported = set(re.findall(r"\bT (cb_\w+)$", nm, re.M))
    assert declared <= exported, declared - exported
    for name in declared:
        assert hasattr(lib, name)


def test_sass_is_sm100a_tcgen05(lib):
    out = subprocess.run(["cuobjdump", "-sass", str(_capi.LIB_PATH)], capture_output=True,
                         text=True).stdout
    if not out:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in subprocess.run(["cuobjdump", "-lelf", str(_capi.LIB_PATH)],
                                       capture_output=True, text=True).stdout
    for mnemonic in ("UTCHMMA", "UTMALDG", "LDTM"):
        assert mnemonic in out, mnemonic
    assert "UTCHMMA.2CTA" in out and "IM2COL" in out


def test_version_and_split_kdim(lib):
    assert lib.cb_version() == 1
    assert [_capi.split_kdim(k) for k in (0, 1, 64, 65, 147)] == [0, 64, 64, 128, 192]


def _shape(lib, d):
    oh, ow = ctypes.c_int32(), ctypes.c_int32()
    _capi.check(lib.cb_output_shape(ctypes.byref(_capi.cdesc(d)), ctypes.byref(oh), ctypes.byref(ow)))
    return oh.value, ow.value


def test_output_shape_matches_descriptor(lib):
    for kw in (dict(in_h=224, in_w=224, k_h=7, k_w=7, stride_h=2, stride_w=2, pad_h=3, pad_w=3),
               dict(in_h=9, in_w=8, k_h=3, k_w=3, dil_h=2, dil_w=1, stride_h=2, pad_h=1),
               dict(in_h=3, in_w=3, k_h=3, k_w=3)):
        d = ConvDescriptor(batch=1, in_channels=4, out_channels=4, **kw)
        assert _shape(lib, d) == output_shape(d)


def test_invalid_descriptors_raise_reference_types(lib):
    bad = _capi.CbConvDesc(1, 4, 2, 2, 4, 5, 5, 1, 1, 0, 0, 1, 1, 1, 0)  # kernel does not fit
    oh, ow = ctypes.c_int32(), ctypes.c_int32()
    with pytest.raises(InvalidDescriptorError, match="does not fit"):
        _capi.check(lib.cb_output_shape(ctypes.byref(bad), ctypes.byref(oh), ctypes.byref(ow)))
    bad = _capi.CbConvDesc(1, 6, 8, 8, 4, 3, 3, 1, 1, 0, 0, 1, 1, 4, 0)  # groups do not divide
    with pytest.raises(InvalidDescriptorError):
        _capi.check(lib.cb_output_shape(ctypes.byref(bad), ctypes.byref(oh), ctypes.byref(ow)))


def test_sconv_rejects_groups_and_dilation(lib):
    for kw in (dict(groups=2), dict(dil_h=2, dil_w=2)):
        d = ConvDescriptor(batch=1, in_channels=4, in_h=9, in_w=9, out_channels=4, k_h=3, k_w=3, **kw)
        sp = _capi.CbSlicePlan()
        with pytest.raises(_capi.UnsupportedDescriptorError, match="groups == 1 and dilation == 1"):
            _capi.check(lib.cb_sconv_plan(ctypes.byref(_capi.cdesc(d)), 64, ctypes.byref(sp)))


def test_sconv_plan_and_ranges(lib):
    d = ConvDescriptor(batch=3, in_channels=8, in_h=10, in_w=10, out_channels=4, k_h=3, k_w=3,
                       pad_h=1, pad_w=1)
    cd = _capi.cdesc(d)
    sp = _capi.CbSlicePlan()
    _capi.check(lib.cb_sconv_plan(ctypes.byref(cd), 30, ctypes.byref(sp)))
    assert (sp.band_rows, sp.num_slices) == (3, 3 * 4)  # ceil(10/3) bands per image
    jb, jc = ctypes.c_int64(), ctypes.c_int64()
    covered = 0
    for first in range(sp.num_slices):
        _capi.check(lib.cb_sconv_range(ctypes.byref(cd), ctypes.byref(sp), first, 1,
                                       ctypes.byref(jb), ctypes.byref(jc)))
        assert jb.value == covered  # slices tile the pixel range contiguously
        covered += jc.value
    assert covered == 3 * 100
    with pytest.raises(InvalidDescriptorError):
        _capi.check(lib.cb_sconv_range(ctypes.byref(cd), ctypes.byref(sp), 11, 2,
                                       ctypes.byref(jb), ctypes.byref(jc)))


def test_workspace_and_layouts(lib):
    from paper_2407_10730_b200 import algos
    from paper_2407_10730_b200.configs import CONFIGS
    d = CONFIGS["cfg4"]
    n = ctypes.c_size_t()
    _capi.check(lib.cb_workspace_bytes(ctypes.byref(_capi.cdesc(d)), 0, None, ctypes.byref(n)))
    assert n.value == 4 * 2304 * 25088  # the im2col matrix
    lay = algos.fused_layout(d, "tc3xbf16")
    assert lay["path"] == 1 and lay["chunk_bytes"] == 128 and lay["weight_cols"] == 2304
    assert lay["workspace_bytes"] >= 2 * 2 * 128 * 196 * 256  # NHWC hi + lo bf16
    lay3 = algos.fused_layout(CONFIGS["cfg3"], "tc3xtf32")  # the direct kernel, tf32 words
    assert lay3["path"] == 2 and lay3["workspace_bytes"] == 0 and lay3["weight_cols"] == 192
    c8 = ConvDescriptor(batch=2, in_channels=8, in_h=32, in_w=32, out_channels=16, k_h=3, k_w=3,
                        pad_h=1, pad_w=1)  # no compile-time layout: the tf32 split keeps K0 + K6
    lay8 = algos.fused_layout(c8, "tc3xtf32")
    assert lay8["path"] == 1 and lay8["chunk_bytes"] == 32  # 8 channels of 4-byte tf32 words
    assert algos.fused_layout(c8, "tc3xbf16")["path"] == 2
    # depthwise with one channel per group cannot use 16-byte chunks: gather path
    dw = ConvDescriptor(batch=1, in_channels=8, in_h=9, in_w=9, out_channels=8, k_h=3, k_w=3,
                        groups=8)
    assert algos.fused_layout(dw, "tc3xbf16")["path"] == 0
    plan = algos.fused_plan(d, "tc3xbf16")
    assert plan["block_m"] in (128, 256) and plan["ctas"] <= 148
    assert algos.plan_tiles(d, "ffma")["block_n"] == 64


def test_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2407_10730_b200 import algos
    from paper_2407_10730_b200.descriptor import ConvDescriptor as D
    import numpy as np
    d = D(batch=1, in_channels=1, in_h=4, in_w=4, out_channels=1, k_h=3, k_w=3)
    inp = algos.ConvInputs(desc=d, input=np.zeros((1, 1, 4, 4), np.float32),
                           weights=np.zeros((1, 1, 3, 3), np.float32))
    with pytest.raises(_capi.ConvB200Error, match="no CPU fallback"):
        algos.conv_fused(inp)


def test_fused_layout_paths(lib):
    """Host-side layout choices of the fused conv (cb_fused_layout_query, no GPU needed):
    K7 for few channels, tap stacking for few output channels, the folded layout, and the
    'auto' variant rule."""
    from paper_2407_10730_b200 import algos
    from paper_2407_10730_b200.configs import CONFIGS
    k7 = algos.fused_layout(CONFIGS["cfg3"], "tc3xbf16")  # C=3 stem: direct TMEM kernel
    assert k7["path"] == 2 and k7["workspace_bytes"] == 0 and k7["weight_cols"] == 192
    full = ConvDescriptor(batch=1, in_channels=128, in_h=12, in_w=12, out_channels=8, k_h=3,
                          k_w=3, pad_h=1, pad_w=1)  # R*S*K = 72 <= 256: all taps stacked
    lay = algos.fused_layout(full, "tc3xbf16")
    assert lay["path"] == 1 and lay["weight_rows"] == 9 * 8 and lay["weight_cols"] == 128
    assert lay["workspace_bytes"] >= 9 * 8 * 12 * 12 * 4  # + the stacked planes Y'
    row = ConvDescriptor(batch=1, in_channels=64, in_h=19, in_w=21, out_channels=32, k_h=7,
                         k_w=7, pad_h=3, pad_w=3)  # S*K = 224: the 7 horizontal taps stacked
    assert algos.fused_layout(row, "tc3xbf16")["weight_rows"] == 7 * 32
    fold = ConvDescriptor(batch=1, in_channels=24, in_h=20, in_w=20, out_channels=64, k_h=5,
                          k_w=5, pad_h=2, pad_w=2)  # 25 taps of 32 -> 5 folded rows of 120
    assert algos.fused_layout(fold, "tc3xbf16")["k_blocks"] == 10
    assert algos.resolve_variant(CONFIGS["cfg1"], "auto") == "tc3xbf16"
    assert algos.resolve_variant(CONFIGS["cfg2a"], "auto") == "ffma"
    assert algos.resolve_variant(CONFIGS["cfg4"], "tc3xtf32") == "tc3xtf32"


def test_fused_tile_plans(lib):
    """K6 tile plans (cb_fused_plan_tiles, host arithmetic; 148 SMs assumed without a GPU):
    CTA pairs with a tail split on the big grid (cfg4: 98 pair tiles on 74 pairs, the 24 tail
    tiles in 3 K parts -> 74 + 72 items on 148 CTAs), single CTAs and no split on short grids
    whose tiles are too short for the fixup to pay (cfg1, cfg2b), a split where it pays
    (cfg2a: 8 tiles x 9 parts), and a huge reduction on few tiles cut into up to 16 K parts
    with CTA pairs (C=2048 7x7 at 56x56: 13 pair tiles x 5 parts)."""
    from paper_2407_10730_b200 import algos
    from paper_2407_10730_b200.configs import CONFIGS
    p4 = algos.fused_plan(CONFIGS["cfg4"], "tc3xbf16")
    assert (p4["block_m"], p4["block_n"], p4["m_tiles"], p4["ctas"]) == (256, 256, 98, 148)
    for name in ("cfg1", "cfg2b"):
        p = algos.fused_plan(CONFIGS[name], "tc3xbf16")
        assert p["block_m"] == 128 and p["ctas"] == p["m_tiles"] * p["n_tiles"] == 25, (name, p)
    p2a = algos.fused_plan(CONFIGS["cfg2a"], "tc3xbf16")
    assert p2a["block_m"] == 128 and p2a["m_tiles"] * p2a["n_tiles"] == 8 and p2a["ctas"] == 72
    from paper_2407_10730_b200.descriptor import parse_key
    big = algos.fused_plan(parse_key("n1_c2048x56x56_f256x7x7_s1x1_p3x3_d1x1_g1_b0"), "tc3xbf16")
    assert (big["block_m"], big["m_tiles"], big["ctas"]) == (256, 13, 130), big


@pytest.mark.parametrize("key,mixed", [
    ("n16_c3x224x224_f64x7x7_s2x2_p3x3_d1x1_g1_b0", True),    # cfg3: pairs + singles, no pad taps
    ("n2_c3x32x32_f16x3x3_s2x2_p1x1_d1x1_g1_b0", True),
    ("n2_c3x32x32_f16x5x5_s2x2_p2x2_d1x1_g1_b0", True),
    ("n2_c4x32x32_f32x3x3_s2x2_p1x1_d1x1_g1_b0", True),
    ("n2_c4x32x32_f32x7x7_s2x2_p3x3_d1x1_g1_b0", True),
    ("n2_c3x32x32_f16x3x3_s1x1_p1x1_d1x1_g1_b0", False),      # odd stride: plain OIHW order
    ("n2_c8x32x32_f16x3x3_s2x2_p1x1_d1x1_g1_b0", False),      # no compile-time layout: plain
])
def test_k7_reduction_map_is_a_permutation(lib, key, mixed):
    """cb_fused_reduction_map (host arithmetic): K7's reduction layout covers every (c, r, s)
    tap exactly once; the mixed layout (even horizontal stride, odd S) has no pad taps inside
    rows, keeps each aligned tap pair (k even, k + 1) on adjacent window columns of one
    (c, r) row, and pairs the rows' single taps two rows at a time."""
    from paper_2407_10730_b200 import algos
    from paper_2407_10730_b200.descriptor import parse_key
    d = parse_key(key)
    assert algos.fused_layout(d, "tc3xbf16")["path"] == 2
    m = algos.fused_reduction_map(d)
    crs = d.in_channels * d.k_h * d.k_w
    taps = [v for v in m if v >= 0]
    assert sorted(taps) == list(range(crs))
    if not mixed:
        assert m == list(range(crs))
        return
    S, nr = d.k_w, d.in_channels * d.k_h
    assert len(m) == crs + (nr & 1)             # one zero element after an odd last row
    assert all(v >= 0 for v in m[:crs - 1])
    singles = 0
    for k in range(0, len(m) - 1, 2):
        a, b = m[k], m[k + 1]
        if a >= 0 and b >= 0 and a // S == b // S:
            assert b == a + 1                   # one LDS.64 of two adjacent columns
        else:
            singles += 1                        # two rows' single taps (or single + zero)
            if b >= 0:
                assert b // S == a // S + 1 and b % S == a % S
    assert singles == (nr + 1) // 2
    assert algos.fused_layout(d, "tc3xbf16")["weight_cols"] == _capi.load().cb_split_kdim(len(m))
    assert algos.fused_reduction_map(d, "tc3xtf32") == m  # the tf32 kernels use the same order
