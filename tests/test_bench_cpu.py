"""bench.py contract pieces that run without a GPU: the reference arm (the ported
reference CPU algorithm) prints one valid JSON line; roofline arithmetic."""

from __future__ import annotations

import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--steps",
                          "1", "--warmup", "0", "--cpu-seconds", "0.3"], capture_output=True,
                         text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["unit"] == "GFLOP/s" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] in ("reference", "port")
    assert line["cpu_baseline"]["cores"] >= 1 and line["cpu_baseline"]["host"]["cpu_count"] >= 1
    if (ROOT / "baseline" / "_ref" / "convbench").exists():
        assert line["cpu_baseline"]["kind"] == "reference"  # the unmodified reference ran
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["higher_is_better"] is True
    assert line["metric"] == json.loads((ROOT / "BASELINE.json").read_text())["metric"]


def test_roofline_arithmetic():
    from paper_2407_10730_b200.configs import CONFIGS, conv_bytes, pack_bytes
    from paper_2407_10730_b200.roofline import conv_roofline
    peaks = {"hbm_gbs": 8000.0, "bf16_tflops": 1657.6, "bf16_tflops_sustained": 1403.3,
             "source": "test"}
    r4 = conv_roofline(CONFIGS["cfg4"], "tc3xtf32", peaks)
    assert r4["flops"] == 29_595_009_024 and r4["bound"] == "tensor"
    assert abs(r4["t_compute_s"] * 1e6 - 107.1) < 0.2  # 3xTF32 = bf16/6
    assert conv_bytes(CONFIGS["cfg4"]) == 53_739_520
    assert pack_bytes(CONFIGS["cfg3"]) == 4 * (16 * 3 * 224 * 224 + 147 * 16 * 112 * 112)
    r2b = conv_roofline(CONFIGS["cfg2b"], "tc3xtf32", peaks)
    assert r2b["bound"] == "hbm"


def test_bench_gpus_flag_starts_the_ranks():
    """`bench.py --gpus 2` with no torchrun environment starts 2 ranks through the shared
    launcher (gloo in --dry-run); rank 0 prints one line for the whole job, strong scaling
    splits the global batch of 128."""
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--dry-run",
                          "--steps", "2", "--warmup", "1"], capture_output=True, text=True,
                         timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(l) for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    line = lines[0]
    assert line["n_gpus"] == 2 and line["scaling"] == "strong" and line["dry_run"] is True
    assert line["config"]["global_batch"] == 128 and line["config"]["images_over_ranks"] == 128
    assert line["config"]["per_gpu_batch"] == 64


def test_bench_rejects_world_size_mismatch():
    import os
    env = dict(os.environ, WORLD_SIZE="4", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--dry-run"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT, env=env)
    assert out.returncode != 0 and "WORLD_SIZE=4" in out.stderr
