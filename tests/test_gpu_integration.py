"""The unmodified reference package driving the B200 path.

`install()` swaps the drop-ins into the reference's own `convbench.harness`; the
reference's CLI then runs main, baseline and correctness sweeps of a convolution set on
the GPU and writes its own results CSVs, which its own `report` command joins.  The
reference comes from baseline/_ref only (the pip --target install that travels with the
repo); nothing here reads /root/reference."""

from __future__ import annotations

import csv

import numpy as np
import pytest

from oracle import conv_oracle as orc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cb():
    from refpkg import reference
    mod = reference(allow_source=False)
    if mod is None:
        pytest.skip("reference convbench not installed in baseline/_ref")
    return mod


def _descs(cb):
    D = cb.descriptor.ConvDescriptor
    return [D(batch=1, in_channels=64, in_h=56, in_w=56, out_channels=64, k_h=3, k_w=3,
              pad_h=1, pad_w=1),                                              # cfg1
            D(batch=1, in_channels=128, in_h=28, in_w=28, out_channels=256, k_h=3, k_w=3,
              stride_h=2, stride_w=2, pad_h=1, pad_w=1),                       # cfg2a
            D(batch=2, in_channels=16, in_h=13, in_w=11, out_channels=24, k_h=5, k_w=3,
              pad_h=2, pad_w=1, has_bias=True),                                # rectangular, bias
            D(batch=1, in_channels=32, in_h=14, in_w=14, out_channels=32, k_h=3, k_w=3,
              pad_h=1, pad_w=1, groups=4)]                                     # grouped


def test_reference_cli_runs_on_the_gpu(cb, tmp_path):
    from paper_2407_10730_b200.harness import install
    cs = cb.convset.ConvSet()
    for d in _descs(cb):
        cs.insert_unique(d)
    path = tmp_path / "set.csv"
    cs.save_csv(path)
    undo = install(cb.harness)
    try:
        outs = {}
        for mode in ("main", "baseline", "correctness"):
            outs[mode] = tmp_path / f"results_{mode}.csv"
            rc = cb.cli.main(["run", "--convset", str(path), "--mode", mode, "--warmups", "1",
                              "--runs", "2", "--out", str(outs[mode])])
            assert rc == 0, mode
    finally:
        undo()
    rows = {m: list(csv.DictReader(open(p))) for m, p in outs.items()}
    assert len(rows["main"]) == 4
    status = {r["key"]: r["status"] for r in rows["main"]}
    assert sorted(status.values()) == ["ok", "ok", "ok", "skipped_unsupported"]  # SConv: groups
    assert all(r["status"] == "ok" for r in rows["baseline"])
    assert all(float(r["in_microkernel_ns_mean"]) > 0 for r in rows["baseline"])
    for r in rows["correctness"]:
        if r["status"] == "ok":
            assert float(r["correctness_max_rel_err"]) <= 1e-4, r["key"]
    # the reference report joins the GPU results unchanged
    rc = cb.cli.main(["report", "--main", str(outs["main"]), "--baseline", str(outs["baseline"]),
                      "--out-speedup", str(tmp_path / "sp.csv"),
                      "--out-breakdown", str(tmp_path / "bd.csv")])
    assert rc in (0, None)
    assert len(list(csv.DictReader(open(tmp_path / "sp.csv")))) == 3


def test_reference_run_single_matches_the_oracle(cb):
    """run_single through the reference harness with the drop-ins installed; the drop-ins'
    outputs for the reference's own make_inputs data match the float64 oracle."""
    from paper_2407_10730_b200 import algos
    from paper_2407_10730_b200.harness import install
    undo = install(cb.harness, main="fused")
    try:
        for d in _descs(cb)[:3]:
            for mode in ("main", "baseline"):
                o = cb.harness.run_single(d, cb.harness.RunConfig(mode=mode, warmups=1, runs=3))
                assert o.status == "ok", (mode, o.detail)
                assert o.stats.operation_ns_mean > 0
            inp = cb.harness.make_inputs(d, cb.harness.RunConfig())
            ref = orc.conv_direct_naive(d, inp.input, inp.weights, inp.bias)
            for fn in (cb.harness.conv_main_blocked_direct, cb.harness.conv_baseline_im2col_gemm):
                y = fn(inp, cb.timing.PhaseLedger())
                assert isinstance(y, np.ndarray) and y.dtype == np.float32
                assert orc.normalized_max_err(y, ref, orc.reduction_len(d)) <= 1e-4
        assert algos._INPUT_CACHE  # inputs were uploaded once and reused
    finally:
        undo()
    assert not algos._INPUT_CACHE_ON
