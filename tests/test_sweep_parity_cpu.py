"""The config-5 parity checker (tests/sweep_parity.py) on CPU: the worker pool regenerates
inputs, computes the float64 oracle and scores outputs handed to it as arrays."""

from __future__ import annotations

import csv
from pathlib import Path

import numpy as np

from oracle import conv_oracle as orc
from paper_2407_10730_b200.descriptor import ConvDescriptor

ROOT = Path(__file__).resolve().parent.parent


def _mod():
    import sweep_parity  # tests/ is on sys.path (conftest); spawned workers import it by name
    return sweep_parity


def test_oracle_checker_scores_outputs(tmp_path):
    sp = _mod()
    d1 = ConvDescriptor(batch=1, in_channels=8, in_h=9, in_w=11, out_channels=6, k_h=3, k_w=3,
                        stride_h=2, stride_w=1, pad_h=1, pad_w=1)
    d2 = ConvDescriptor(batch=1, in_channels=4, in_h=7, in_w=7, out_channels=5, k_h=1, k_w=1)
    chk = sp.OracleChecker(data_seed=0, workers=2, pending=1, spool=str(tmp_path))
    x, w, b = orc.make_inputs(d1, 0)
    good = orc.conv_direct_naive(d1, x, w, b)
    bad = good.copy()
    bad[0, 2, 1, 3] += 1.0
    chk.check(d1, None, [(0, "fused", good), (0, "main", bad), (7, "fused", good)])
    x2, w2, b2 = orc.make_inputs(d2, 0)
    chk.check(d2, None, [(3, "baseline", orc.conv_direct_naive(d2, x2, w2, b2)[:, :4])])
    res = chk.finish()
    assert res["0:fused"]["err"] < 1e-7 and res["7:fused"]["err"] < 1e-7
    assert abs(res["0:main"]["err"] - 1.0 / np.sqrt(8 * 9)) < 1e-6
    assert res["3:baseline"]["err"] == float("inf") and "shape" in res["3:baseline"]["note"]
    assert not list(Path(chk.dir).glob("*.npy"))  # spool cleaned up
    s = chk.summarize("fused", [(0, "k0", "ok"), (7, "k0", "ok"), (9, "k9", "failed")], res)
    assert s["checked"] == 2 and s["unchecked"] == 1 and s["over_gate"] == 0
    s = chk.summarize("main", [(0, "k0", "ok")], res)
    assert s["over_gate"] == 1 and s["worst_op"]["index"] == 0
    descs = {0: d1, 3: d2, 7: d1}
    chk.write_table(tmp_path / "p.csv", descs, res)
    rows = list(csv.DictReader(open(tmp_path / "p.csv")))
    assert [(r["index"], r["mode"]) for r in rows] == [("0", "fused"), ("0", "main"),
                                                       ("3", "baseline"), ("7", "fused")]


def test_channel_subset_oracle_for_large_ops(tmp_path):
    """Ops above the oracle budget are checked on a seeded subset of output channels (every
    pixel of each): the subset oracle equals those channels of the full oracle."""
    sp = _mod()
    d = ConvDescriptor(batch=1, in_channels=16, in_h=10, in_w=10, out_channels=40, k_h=3, k_w=3,
                       pad_h=1, pad_w=1)
    from paper_2407_10730_b200.descriptor import flop_count
    assert sp.oracle_channels(d, flop_count(d)) is None
    ch = sp.oracle_channels(d, flop_count(d) / 10)
    assert len(ch) == 8 and (np.diff(ch) > 0).all()
    assert np.array_equal(ch, sp.oracle_channels(d, flop_count(d) / 10))  # seeded
    x, w, b = orc.make_inputs(d, 0)
    y = orc.conv_direct_naive(d, x, w, b)
    y_bad = y.copy()
    y_bad[0, ch[3], 4, 4] += 0.5
    np.save(tmp_path / "a.npy", y)
    np.save(tmp_path / "b.npy", y_bad)
    res = sp._check_job(d, 0, [(0, "fused", str(tmp_path / "a.npy")),
                               (1, "fused", str(tmp_path / "b.npy"))], ch)
    assert res[0][2] < 1e-7 and "8/40 channels" in res[0][4]
    assert abs(res[1][2] - 0.5 / np.sqrt(16 * 9)) < 1e-6
