"""Summarise ncu captures (gpurun_out/prof/) into committed evidence under profiles/.

    python tools/ncu_summary.py gpurun_out/prof r01

Writes profiles/<tag>_launches.csv (per-kernel share of the bench command's launch list),
profiles/<tag>_ncu_<kernel>.txt (key metrics of each full capture) and
profiles/ncu_summary.json (per-launch DRAM traffic that bench.py reports as
roofline.traffic).
"""

from __future__ import annotations

import csv
import io
import json
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
KEYS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "dram__bytes_read.sum",
    "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__m_xbar2l1tex_read_bytes.sum", "l1tex__m_xbar2l1tex_read_bytes.sum.per_second",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__shared_mem_per_block_dynamic", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed_op_tma_ld.sum", "sm__inst_executed.sum",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smsp__inst_executed_op_shared_ld.sum",
    "smsp__inst_executed_op_shared_st.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "smsp__pcsamp_warps_issue_stalled_long_scoreboard", "smsp__pcsamp_warps_issue_stalled_short_scoreboard",
    "smsp__pcsamp_warps_issue_stalled_wait", "smsp__pcsamp_warps_issue_stalled_barrier",
    "smsp__pcsamp_warps_issue_stalled_no_instructions", "smsp__pcsamp_warps_issue_stalled_math_pipe_throttle",
    "smsp__pcsamp_warps_issue_stalled_lg_throttle", "smsp__pcsamp_warps_issue_stalled_mio_throttle",
    "smsp__pcsamp_sample_count",
]


SHORT = {"conv_tma_kernel": "conv_tma", "act_split_nhwc_kernel": "act_split", "act_split_wide_kernel": "act_split",
         "act_fold_split_kernel": "act_fold_split", "weight_split_taps_kernel": "weight_split_taps",
         "im2col_band_kernel": "im2col_band", "im2col_kernel": "im2col_kernel",
         "conv_tc_kernel": "conv_tc", "conv_ts_kernel": "conv_ts", "gemm_ts_kernel": "gemm_ts",
         "tap_sum_kernel": "tap_sum", "unpack_rows_kernel": "unpack"}


def raw_metrics(rep: Path) -> list[dict]:
    """One dict per profiled kernel launch in the report."""
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        m = {"kernel": vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else ""}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                m[k] = (vals[i], units[i])
        res.append(m)
    return res


def short_name(kernel: str) -> str:
    base = kernel.replace("void ", "").split("(")[0].split("<")[0].split("::")[-1]
    if base == "conv_ts_kernel":  # the last template argument: 1 / true = bf16 pairs, 0 / false = tf32 words
        args = kernel.split("(")[0].split("<")[-1].split(">")[0].replace(" ", "").replace("(bool)", "").split(",")
        if len(args) >= 4 and args[-1] in ("0", "false"):
            return "conv_ts_tf32"
    return SHORT.get(base, base)


def to_bytes(v, unit) -> float:
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    return float(v.replace(",", "")) * scale


def main(src: str, tag: str) -> None:
    src_p = Path(src)
    prof = ROOT / "profiles"
    prof.mkdir(exist_ok=True)
    # launch list -> per-kernel share
    rows = list(csv.reader(open(src_p / "launches.csv")))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, mi = h.index("Kernel Name"), h.index("Metric Value")
    agg = defaultdict(list)
    for r in rows[hi + 1:]:
        if len(r) > mi:
            agg[r[ki].split("(")[0]].append(float(r[mi].replace(",", "")))
    total = sum(sum(v) for v in agg.values())
    with open(prof / f"{tag}_launches.csv", "w") as f:
        f.write("kernel,launches,mean_ns,total_ns,share\n")
        for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
            f.write(f"\"{k}\",{len(v)},{sum(v) / len(v):.0f},{sum(v):.0f},{sum(v) / total:.4f}\n")
    summary = {}
    sj = prof / "ncu_summary.json"
    if sj.exists():
        summary = json.loads(sj.read_text())
    for rep in sorted(src_p.glob("full_*.ncu-rep")):
      for m in raw_metrics(rep):
        name = short_name(m.get("kernel", "")) or rep.stem.replace("full_", "")
        lines = [f"# ncu --set full --clock-control none, {tag}: {m.get('kernel', '')[:160]}"]
        for k in KEYS:
            if k in m:
                lines.append(f"{k:70s} {m[k][0]:>16s} {m[k][1]}")
        (prof / f"{tag}_ncu_{name}.txt").write_text("\n".join(lines) + "\n")
        rd = to_bytes(*m["dram__bytes_read.sum"]) if "dram__bytes_read.sum" in m else None
        wr = to_bytes(*m["dram__bytes_write.sum"]) if "dram__bytes_write.sum" in m else None
        summary[name] = {"kernel": m.get("kernel", "")[:160],
                         "duration_us": float(m["gpu__time_duration.sum"][0].replace(",", ""))
                         if m["gpu__time_duration.sum"][1] == "us" else None,
                         "dram_bytes": (rd or 0) + (wr or 0), "dram_read": rd, "dram_write": wr,
                         "capture": f"profiles/{tag}_ncu_{name}.txt"}
    # bench.py looks traffic up as "<config>/<variant>"
    if "conv_tma" in summary:
        summary["cfg4/tc3xbf16"] = summary["conv_tma"]
    sj.write_text(json.dumps(summary, indent=1) + "\n")
    print((prof / f"{tag}_launches.csv").read_text())
    print(json.dumps(summary, indent=1))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/prof", sys.argv[2] if len(sys.argv) > 2 else "r01")
