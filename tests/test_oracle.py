"""Pin the CPU oracle (oracle/) against golden vectors produced by the reference itself
(tests/golden/make_golden.py): input generation, im2col bytes, the float64 oracle and the
ported reference algorithms (bit-exact outputs and phase call counts).  CPU only."""

from __future__ import annotations

import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

from oracle import conv_oracle as orc
from oracle import reference_port as rp
from paper_2407_10730_b200.descriptor import parse_key

GOLD = Path(__file__).resolve().parent / "golden"


def sha(a) -> str:
    return "" if a is None else hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def corpus():
    z = np.load(GOLD / "corpus.npz")
    return json.loads(str(z["meta"])), z


class CountLedger:
    def __init__(self):
        self.calls = [0] * 7

    def start(self, p):
        pass

    def update(self, p):
        self.calls[int(p)] += 1


def test_corpus_inputs_and_im2col(corpus):
    rows, _ = corpus
    assert len(rows) >= 30
    for r in rows:
        d = parse_key(r["key"])
        x, w, b = orc.make_inputs(d, seed=0)
        assert (sha(x), sha(w), sha(b)) == (r["x"], r["w"], r["b"]), r["key"]
        assert sha(orc.im2col(d, x)) == r["im2col"], r["key"]


def test_corpus_oracle_outputs(corpus):
    rows, z = corpus
    for i, r in enumerate(rows):
        d = parse_key(r["key"])
        x, w, b = orc.make_inputs(d, seed=0)
        want = z[f"naive_{i}"]
        got = orc.conv_direct_naive(d, x, w, b)
        assert sha(got) == r["naive"] and np.array_equal(got, want), r["key"]
        # the float64 im2col GEMM oracle agrees to fp32 rounding
        assert orc.normalized_max_err(orc.conv_im2col64(d, x, w, b), want,
                                      orc.reduction_len(d)) < 1e-6
        # the banded float64 oracle of the sweep parity run, with bands of 1-2 rows
        for cap in (1, 1 << 12):
            got64 = orc.conv_banded64(d, x, w, b, max_cols_bytes=cap)
            assert orc.normalized_max_err(got64, want, orc.reduction_len(d)) < 1e-6, r["key"]
        if i < 6:  # literal loops on the smallest shapes (reference tests/oracles.py:43-80)
            assert orc.normalized_max_err(orc.conv_loops(d, x, w, b), want,
                                          orc.reduction_len(d)) < 1e-6


def test_corpus_reference_port_bit_exact(corpus):
    rows, _ = corpus
    n_main = 0
    for r in rows:
        d = parse_key(r["key"])
        x, w, b = orc.make_inputs(d, seed=0)
        led = CountLedger()
        assert sha(rp.conv_baseline_im2col_gemm(d, x, w, b, led)) == r["baseline"], r["key"]
        assert led.calls == r["baseline_calls"], r["key"]
        if r["main"] is None:
            with pytest.raises(ValueError):
                rp.conv_main_blocked_direct(d, x, w, b)
            continue
        led = CountLedger()
        assert sha(rp.conv_main_blocked_direct(d, x, w, b, led)) == r["main"], r["key"]
        assert led.calls == r["main_calls"], r["key"]
        n_main += 1
    assert n_main >= 12


@pytest.mark.parametrize("name", ["cfg1", "cfg2a", "cfg2b", "cfg3", "cfg4"])
def test_baseline_configs_pinned(name):
    from paper_2407_10730_b200.configs import CONFIGS
    z = np.load(GOLD / "configs.npz")
    meta = json.loads(str(z["meta"]))[name]
    d = CONFIGS[name]
    assert parse_key(meta["key"]) == d
    x, w, b = orc.make_inputs(d, seed=0)
    assert (sha(x), sha(w)) == (meta["x"], meta["w"])
    y = orc.conv_im2col64(d, x, w, b)
    assert list(y.shape) == meta["shape"]
    vals = y.reshape(-1)[z[f"{name}_idx"]]
    err = orc.normalized_max_err(vals, z[f"{name}_val"], orc.reduction_len(d))
    assert err < 1e-6, err
    y64 = y.astype(np.float64)
    assert abs(y64.sum() - meta["sum"]) <= 1e-6 * meta["sumsq"] ** 0.5 * 10
    assert abs((y64 ** 2).sum() / meta["sumsq"] - 1) < 1e-6


def test_slice_pack_is_im2col_columns():
    from paper_2407_10730_b200.descriptor import ConvDescriptor
    d = ConvDescriptor(batch=2, in_channels=3, in_h=9, in_w=7, out_channels=4, k_h=3, k_w=3,
                       pad_h=1, pad_w=1, stride_h=2, stride_w=1)
    x, _, _ = orc.make_inputs(d, 0)
    oh, ow = orc.output_shape(d)
    cols = orc.im2col(d, x)
    whole = orc.slice_pack(d, x, oh, 0, d.batch)  # one slice per image
    assert np.array_equal(whole.reshape(cols.shape), cols)
    # 2-row bands (3 per image): slices 1..3 = image 0 rows 2-4 and image 1 rows 0-1, one
    # column block across the image boundary
    part = orc.slice_pack(d, x, 2, 1, 3)
    assert np.array_equal(part.reshape(cols.shape[0], -1), cols[:, 2 * ow: oh * ow + 2 * ow])


def test_parity_metrics():
    a = np.array([1.0, 2.0], np.float32)
    assert orc.normalized_max_err(a, a, 9) == 0.0
    assert orc.normalized_max_err(a + 3e-4, a, 9) == pytest.approx(1e-4, rel=1e-2)
    assert orc.normalized_max_err(np.array([np.nan]), np.array([0.0]), 1) == float("inf")
    assert orc.reference_allclose_err(a, a) == 0.0
