"""Results-CSV schema (reference report.py:21-27) and the config-5 sweep plumbing (CPU)."""

from __future__ import annotations

import csv
import importlib.util
from pathlib import Path

from paper_2407_10730_b200 import configs, report
from paper_2407_10730_b200.harness import RunOutcome
from paper_2407_10730_b200.timing import TimingReport, aggregate, Phase

ROOT = Path(__file__).resolve().parent.parent
STEMS = ["pre_analysis", "pre_reorder", "in_tiling", "in_packing", "in_microkernel",
         "in_unpacking", "post_reorder"]


def _sweep_mod():
    spec = importlib.util.spec_from_file_location("sweep_tool", ROOT / "tools" / "sweep.py")
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def test_results_header_is_reference_schema():
    want = ["key", "mode", "status", "runs", "warmups"]
    for s in STEMS:
        want += [f"{s}_ns_mean", f"{s}_ns_min", f"{s}_calls"]
    want += ["operation_ns_mean", "operation_ns_min", "convolution_ns_mean",
             "convolution_ns_min", "correctness_max_rel_err"]
    assert report.RESULTS_HEADER == want


def _report(vals):
    from paper_2407_10730_b200.timing import _report as mk
    return mk(vals, [1 if v else 0 for v in vals])


def test_results_roundtrip(tmp_path):
    stats = aggregate([_report([0, 100, 0, 0, 400, 0, 0]), _report([0, 120, 0, 0, 380, 0, 0])])
    outs = [RunOutcome(key="k1", mode="baseline", runs=2, warmups=1, status="ok", stats=stats),
            RunOutcome(key="k2", mode="baseline", runs=2, warmups=1,
                       status="skipped_unsupported", detail="groups")]
    p = tmp_path / "r.csv"
    report.write_results_csv(outs, p)
    rows = report.read_results_csv(p)
    assert [r.key for r in rows] == ["k1", "k2"]
    assert rows[0].operation_ns_mean == 500.0 and rows[0].operation_ns_min == 480
    assert rows[0].phase_ns_mean[Phase.PRE_REORDER] == 110.0
    assert rows[1].operation_ns_mean is None
    with open(p) as fh:
        assert len(next(csv.reader(fh))) == len(report.RESULTS_HEADER)


def test_stratified_sample_and_lpt_cover_the_sweep():
    sw = _sweep_mod()
    descs = configs.sweep(500, 0)
    a = sw.stratified_sample(descs, 50, 0)
    assert a == sw.stratified_sample(descs, 50, 0) and len(a) == 50 == len(set(a))
    from paper_2407_10730_b200.shard import lpt_assign
    peaks = {"hbm_gbs": 6500.0, "bf16_tflops": 1600.0, "bf16_tflops_sustained": 1400.0}
    cost = [sw.predicted_s(descs[i], peaks) for i in a]
    parts = lpt_assign(cost, 4)
    assert sorted(j for p in parts for j in p) == list(range(len(a)))
    loads = [sum(cost[j] for j in p) for p in parts]
    assert max(loads) <= sum(loads) / 4 + max(cost) + 1e-12


def test_model_op_set_is_valid():
    """configs/model_ops.json (tools/model_ops.py): every layer key parses into a valid
    descriptor, and the unique list covers exactly the layers of all models."""
    import json
    from paper_2407_10730_b200.descriptor import key_of, parse_key
    data = json.loads((ROOT / "configs" / "model_ops.json").read_text())
    layers = [k for m in data["models"].values() for k in m["layers"]]
    assert set(layers) == set(data["unique"]) and len(data["unique"]) >= 300
    for k in data["unique"]:
        assert key_of(parse_key(k)) == k
    assert data["models"]["resnet50"]["layers"][0].startswith("n1_c3x224x224_f64x7x7_s2x2_p3x3")


def test_charts_from_report_csvs(tmp_path):
    """tools/charts.py renders the reference report's speedup and breakdown CSVs as SVG:
    one bar per op (blue >= 1, red < 1), stacked phases per side; byte-identical reruns."""
    import xml.etree.ElementTree as ET
    spec = importlib.util.spec_from_file_location("charts_tool", ROOT / "tools" / "charts.py")
    charts = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(charts)
    sp = tmp_path / "speedup.csv"
    sp.write_text("key,flops,operation_speedup,convolution_speedup\n"
                  "a,10,2.0,1.5\nb,30,0.5,0.8\nc,20,1.0,3.0\n")
    bd = tmp_path / "breakdown.csv"
    cols = ["index", "key", "side"] + [f"{s}_ms" for s in charts.PHASE_STEMS] + ["operation_ms"]
    lines = [",".join(cols)]
    for i in range(2):
        for side in ("main", "baseline"):
            lines.append(",".join([str(i), f"k{i}", side] + ["0.5"] * 7 + ["3.5"]))
    bd.write_text("\n".join(lines) + "\n")
    for args in (["speedup", "--in", str(sp), "--out", str(tmp_path / "s.svg"), "--sort", "by-flops"],
                 ["speedup", "--in", str(sp), "--out", str(tmp_path / "l.svg"), "--log-y",
                  "--scope", "operation"],
                 ["breakdown", "--in", str(bd), "--out", str(tmp_path / "b.svg")]):
        assert charts.main(args) == 0
    s = (tmp_path / "s.svg").read_text()
    root = ET.fromstring(s)
    fills = [e.get("fill") for e in root.iter("{http://www.w3.org/2000/svg}rect")][1:]
    assert fills == [charts.SPEEDUP_COLOR, charts.SPEEDUP_COLOR, charts.SLOWDOWN_COLOR]  # by flops
    ET.fromstring((tmp_path / "l.svg").read_text())
    b = ET.fromstring((tmp_path / "b.svg").read_text())
    assert len(list(b.iter("{http://www.w3.org/2000/svg}rect"))) == 1 + 2 * 2 * 7 + 7
    assert charts.main(["speedup", "--in", str(sp), "--out", str(tmp_path / "s2.svg"),
                        "--sort", "by-flops"]) == 0
    assert (tmp_path / "s2.svg").read_bytes() == (tmp_path / "s.svg").read_bytes()
    (tmp_path / "bad.csv").write_text("key,flops\n")
    assert charts.main(["speedup", "--in", str(tmp_path / "bad.csv"), "--out", str(tmp_path / "x.svg")]) == 1


def test_sweep_gpus_flag_dry_run(tmp_path):
    """`tools/sweep.py --gpus 2 --dry-run` starts 2 ranks through the shared launcher (gloo):
    the LPT partition covers every op exactly once across ranks, rank 0 gathers and writes
    the reference-schema results CSVs and a summary for the whole job."""
    import csv
    import json
    import subprocess
    import sys
    out = tmp_path / "sw"
    r = subprocess.run([sys.executable, str(ROOT / "tools" / "sweep.py"), "--gpus", "2", "--dry-run",
                        "--ops", "120", "--modes", "fused,main", "--out", str(out)],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    summary = json.loads((out / "summary.json").read_text())
    assert summary["world"] == 2 and summary["ops_run"] == 120
    for m in ("fused", "main"):
        rows = list(csv.reader(open(out / f"results_{m}.csv")))[1:]
        assert len(rows) == 120 and all(row[2] == "ok" for row in rows)
        busy = summary["modes"][m]["per_rank_busy_s"]
        assert len(busy) == 2 and min(busy) > 0
