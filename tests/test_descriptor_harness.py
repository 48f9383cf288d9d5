"""Data model and sweep engine on the host (CPU only): descriptor validation / keys /
FLOPs as the reference defines them, seeded inputs pinned to the reference's bytes, the
synthetic sweep generator, drop-in installation into a reference-shaped harness."""

from __future__ import annotations

import hashlib
import json
import types
from pathlib import Path

import numpy as np
import pytest

from paper_2407_10730_b200.descriptor import (ConvDescriptor, InvalidDescriptorError, classify,
                                              flop_count, key_of, output_shape, parse_key)
from paper_2407_10730_b200.harness import RunConfig, install, make_inputs, sweep_shard
from paper_2407_10730_b200.tensor import allclose, normalized_max_err

GOLD = Path(__file__).resolve().parent / "golden"


def D(**kw):
    base = dict(batch=1, in_channels=2, in_h=6, in_w=6, out_channels=3, k_h=3, k_w=3)
    base.update(kw)
    return ConvDescriptor(**base)


def test_descriptor_validation():
    for kw in (dict(batch=0), dict(k_h=0), dict(stride_w=0), dict(groups=0)):
        with pytest.raises(InvalidDescriptorError):
            D(**kw)
    with pytest.raises(InvalidDescriptorError, match="padding"):
        D(pad_h=-1)
    with pytest.raises(InvalidDescriptorError, match="divisible"):
        D(in_channels=3, groups=2, out_channels=4)
    with pytest.raises(InvalidDescriptorError, match="does not fit"):
        D(in_h=2, in_w=2)


def test_shapes_keys_flops_known_answers():
    assert output_shape(D(in_h=224, in_w=224, k_h=7, k_w=7, stride_h=2, stride_w=2, pad_h=3,
                          pad_w=3)) == (112, 112)
    d = D(has_bias=True, groups=1)
    assert parse_key(key_of(d)) == d
    assert key_of(d) == "n1_c2x6x6_f3x3x3_s1x1_p0x0_d1x1_g1_b1"
    one = ConvDescriptor(batch=1, in_channels=1, in_h=1, in_w=1, out_channels=1, k_h=1, k_w=1)
    assert flop_count(one) == 2
    assert flop_count(ConvDescriptor(1, 2, 3, 3, 1, 3, 3)) == 36
    assert flop_count(ConvDescriptor(1, 1, 3, 3, 1, 3, 3, has_bias=True)) == 19
    assert classify(D(k_h=1, k_w=1)).names() == {"pointwise"}
    assert classify(D(in_channels=4, out_channels=4, groups=2, dil_h=2, k_w=1, in_h=9)).names() == \
        {"grouped", "dilated", "rectangular"}


def test_make_inputs_matches_reference_bytes():
    rows = json.loads(str(np.load(GOLD / "corpus.npz")["meta"]))
    sha = lambda a: "" if a is None else hashlib.sha256(a.tobytes()).hexdigest()
    for r in rows[:16]:
        inp = make_inputs(parse_key(r["key"]), RunConfig(seed=0))
        assert (sha(inp.input), sha(inp.weights), sha(inp.bias)) == (r["x"], r["w"], r["b"])
    c = make_inputs(D(has_bias=True), RunConfig(data_gen="constant", constant_value=2.5))
    assert (c.input == 2.5).all() and (c.bias == 2.5).all()


def test_run_config_validation():
    assert (RunConfig().warmups, RunConfig().runs) == (10, 100)
    for kw in (dict(mode="fastest"), dict(data_gen="zeros"), dict(runs=0), dict(warmups=-1)):
        with pytest.raises(ValueError):
            RunConfig(**kw)


def test_conv_inputs_validation():
    from paper_2407_10730_b200.algos import ConvInputs
    d = D()
    x = np.zeros((1, 2, 6, 6), np.float32)
    w = np.zeros((3, 2, 3, 3), np.float32)
    with pytest.raises(ValueError, match="input shape"):
        ConvInputs(desc=d, input=x[:, :1], weights=w)
    with pytest.raises(ValueError, match="weights shape"):
        ConvInputs(desc=d, input=x, weights=w[:, :, :1])
    with pytest.raises(ValueError, match="bias"):
        ConvInputs(desc=D(has_bias=True), input=x, weights=w)
    with pytest.raises(ValueError, match="bias"):
        ConvInputs(desc=d, input=x, weights=w, bias=np.zeros(3, np.float32))


def test_metrics():
    a = np.ones(4, np.float32)
    ok, err = allclose(a, a)
    assert ok and err == 0.0
    ok, err = allclose(a * (1 + 2e-4), a)
    assert not ok and err > 1e-4
    assert normalized_max_err(a + 1e-4, a, 1) == pytest.approx(1e-4, rel=1e-3)


def test_sweep_generator():
    from paper_2407_10730_b200.configs import SWEEP_SIZE, sweep
    s = sweep()
    assert len(s) == SWEEP_SIZE == 9243
    assert s == sweep()  # seeded
    keys = {key_of(d) for d in s}
    assert 2000 < len(keys) < 5000  # duplicates kept as distinct indexed ops
    assert {d.in_h for d in s} == {7, 14, 28, 56, 112, 224}
    assert {d.k_h for d in s} == {1, 3, 5, 7}
    frac3 = sum(d.in_channels == 3 for d in s) / len(s)
    assert 0.03 < frac3 < 0.07
    assert all(d.pad_h == d.k_h // 2 and d.batch == 1 for d in s)


def test_sweep_shard_covers_all():
    from paper_2407_10730_b200.configs import sweep
    s = sweep(500, seed=1)
    parts = [sweep_shard(s, r, 8, cost=flop_count) for r in range(8)]
    allidx = sorted(i for p in parts for i in p)
    assert allidx == list(range(500))
    loads = [sum(flop_count(s[i]) for i in p) for p in parts]
    assert max(loads) <= 1.25 * (sum(loads) / 8) + max(flop_count(d) for d in s)


def test_install_into_reference_shaped_harness():
    """install() rebinds the module globals the reference harness looks up at call time
    (harness.py:99-104,119) and restores them."""
    class RefUnsupported(ValueError):
        pass

    ref = types.SimpleNamespace(conv_main_blocked_direct="m", conv_baseline_im2col_gemm="b",
                                PhaseLedger="L", UnsupportedDescriptorError=RefUnsupported)
    undo = install(ref)
    assert callable(ref.conv_main_blocked_direct) and callable(ref.conv_baseline_im2col_gemm)
    from paper_2407_10730_b200.timing import EventLedger
    assert ref.PhaseLedger is EventLedger
    # ours -> the reference's exception class, so the reference reports skipped_unsupported
    grouped = make_inputs(D(in_channels=4, out_channels=4, groups=2), RunConfig())
    with pytest.raises(RefUnsupported):
        ref.conv_main_blocked_direct(grouped, None)
    undo()
    assert (ref.conv_main_blocked_direct, ref.PhaseLedger) == ("m", "L")
