"""Charts of `convbench report` CSVs without matplotlib.

    python tools/charts.py speedup   --in speedup.csv   --out speedup.svg [--scope operation]
                                     [--sort convset-order|by-speedup|by-flops] [--log-y]
    python tools/charts.py breakdown --in breakdown.csv --out breakdown.svg

The same two figures, inputs and options as the reference renderer
(pkg/tools/src/convbench_tools/charts.py:103-171): a per-operation speedup bar chart with
bars straddling y = 1 (blue >= 1, red < 1), and a side-by-side stacked per-phase time
breakdown (main bar left, baseline bar right, ms).  The reference draws with matplotlib,
which this image lacks; this writes the SVG directly.  Output is a pure function of the
input CSV (fixed geometry, colours, number formatting; no timestamps), so two runs over the
same file are byte-identical, as the reference guarantees for its own output.
"""

from __future__ import annotations

import argparse
import csv
import math
import sys
from html import escape

PHASE_STEMS = ["pre_analysis", "pre_reorder", "in_tiling", "in_packing", "in_microkernel",
               "in_unpacking", "post_reorder"]
PHASE_COLORS = {"pre_analysis": "#8c8c8c", "pre_reorder": "#937860", "in_tiling": "#ccb974",
                "in_packing": "#c44e52", "in_microkernel": "#4c72b0", "in_unpacking": "#55a868",
                "post_reorder": "#8172b3"}
SPEEDUP_COLOR, SLOWDOWN_COLOR = "#4c72b0", "#c44e52"
SCOPES = ("convolution", "operation")
SORTS = ("convset-order", "by-speedup", "by-flops")
W, H = 1000, 400
LEFT, RIGHT, TOP, BOTTOM = 70, 20, 20, 50


class ChartDataError(ValueError):
    """Input CSV is missing required columns or rows."""


def _read_csv(path: str, required: list[str]) -> list[dict[str, str]]:
    with open(path, newline="", encoding="utf-8") as fh:
        reader = csv.DictReader(fh)
        missing = [c for c in required if c not in (reader.fieldnames or [])]
        if missing:
            raise ChartDataError(f"{path}: missing columns {missing}")
        rows = list(reader)
    if not rows:
        raise ChartDataError(f"{path}: no data rows")
    return rows


def _fmt(v: float) -> str:
    return f"{v:.6g}"


class _Svg:
    def __init__(self):
        self.parts = [f'<svg xmlns="http://www.w3.org/2000/svg" width="{W}" height="{H}" '
                      f'viewBox="0 0 {W} {H}" font-family="DejaVu Sans" font-size="9">',
                      f'<rect x="0" y="0" width="{W}" height="{H}" fill="white"/>']

    def rect(self, x, y, w, h, fill):
        if h < 0:
            y, h = y + h, -h
        self.parts.append(f'<rect x="{x:.2f}" y="{y:.2f}" width="{max(w, 0.01):.2f}" '
                          f'height="{h:.2f}" fill="{fill}"/>')

    def line(self, x0, y0, x1, y1, stroke="black", width=0.8, opacity=1.0):
        self.parts.append(f'<line x1="{x0:.2f}" y1="{y0:.2f}" x2="{x1:.2f}" y2="{y1:.2f}" '
                          f'stroke="{stroke}" stroke-width="{width}" stroke-opacity="{opacity}"/>')

    def text(self, x, y, s, anchor="middle", rotate=None, size=9):
        tr = f' transform="rotate({rotate} {x:.2f} {y:.2f})"' if rotate is not None else ""
        self.parts.append(f'<text x="{x:.2f}" y="{y:.2f}" text-anchor="{anchor}" '
                          f'font-size="{size}"{tr}>{escape(s)}</text>')

    def done(self) -> str:
        return "\n".join(self.parts + ["</svg>"]) + "\n"


def _axes(svg: _Svg, ymin: float, ymax: float, log: bool, xlabel: str, ylabel: str):
    """Frame, grid and y ticks; returns value -> pixel y."""
    ph = H - TOP - BOTTOM

    def ty(v: float) -> float:
        if log:
            lo, hi = math.log10(ymin), math.log10(ymax)
            v = math.log10(max(v, ymin))
        else:
            lo, hi = ymin, ymax
        return TOP + ph * (1.0 - (v - lo) / ((hi - lo) or 1.0))
    if log:
        ticks = [10.0 ** e for e in range(math.floor(math.log10(ymin)), math.ceil(math.log10(ymax)) + 1)]
    else:
        step = 10 ** math.floor(math.log10((ymax - ymin) / 5 or 1.0))
        for m in (1, 2, 5, 10):
            if (ymax - ymin) / (step * m) <= 8:
                step *= m
                break
        ticks = [ymin + i * step for i in range(int((ymax - ymin) / step) + 1)]
    for t in ticks:
        y = ty(t)
        if TOP - 0.5 <= y <= H - BOTTOM + 0.5:
            svg.line(LEFT, y, W - RIGHT, y, stroke="#b0b0b0", width=0.5, opacity=0.3)
            svg.text(LEFT - 4, y + 3, _fmt(t), anchor="end")
    svg.line(LEFT, TOP, LEFT, H - BOTTOM)
    svg.line(LEFT, H - BOTTOM, W - RIGHT, H - BOTTOM)
    svg.text((LEFT + W - RIGHT) / 2, H - 12, xlabel)
    svg.text(16, (TOP + H - BOTTOM) / 2, ylabel, rotate=-90)
    return ty


def speedup_svg(input_path: str, scope: str = "convolution", sort: str = "convset-order",
                log_y: bool = False) -> str:
    if scope not in SCOPES or sort not in SORTS:
        raise ValueError(f"scope in {SCOPES}, sort in {SORTS}")
    col = f"{scope}_speedup"
    rows = _read_csv(input_path, ["key", "flops", col])
    data = [(r["key"], int(r["flops"]), float(r[col])) for r in rows]
    if sort == "by-speedup":
        data.sort(key=lambda t: t[2])
    elif sort == "by-flops":
        data.sort(key=lambda t: t[1])
    vals = [t[2] for t in data]
    svg = _Svg()
    ymin = min(min(vals), 1.0)
    ymax = max(max(vals), 1.0)
    if log_y:
        ymin, ymax = ymin / 1.2, ymax * 1.2
    else:
        ymin, ymax = min(0.0, ymin), ymax * 1.05
    ty = _axes(svg, ymin, ymax, log_y, "operation index", f"{scope} speedup (baseline / main)")
    pw = W - LEFT - RIGHT
    slot = pw / max(1, len(vals))
    base = ty(1.0)
    for i, v in enumerate(vals):
        x = LEFT + slot * (i + 0.1)
        svg.rect(x, base, slot * 0.8, ty(v) - base, SPEEDUP_COLOR if v >= 1.0 else SLOWDOWN_COLOR)
    svg.line(LEFT, base, W - RIGHT, base)
    return svg.done()


def breakdown_svg(input_path: str) -> str:
    cols = ["index", "key", "side"] + [f"{s}_ms" for s in PHASE_STEMS] + ["operation_ms"]
    rows = _read_csv(input_path, cols)
    sides: dict[str, dict[int, list[float]]] = {"main": {}, "baseline": {}}
    order: list[int] = []
    for r in rows:
        idx = int(r["index"])
        if r["side"] not in sides:
            raise ChartDataError(f"{input_path}: unknown side {r['side']!r}")
        sides[r["side"]][idx] = [float(r[f"{s}_ms"]) for s in PHASE_STEMS]
        if idx not in order:
            order.append(idx)
    tot = max(sum(v) for s in sides.values() for v in s.values()) if any(sides.values()) else 1.0
    svg = _Svg()
    ty = _axes(svg, 0.0, tot * 1.05 or 1.0, False, "operation index (main left, baseline right)",
               "time (ms)")
    pw = W - LEFT - RIGHT
    slot = pw / max(1, len(order))
    for k, idx in enumerate(order):
        for off, side in ((0.08, "main"), (0.5, "baseline")):
            x = LEFT + slot * (k + off)
            acc = 0.0
            for pi, stem in enumerate(PHASE_STEMS):
                h = sides[side].get(idx, [0.0] * len(PHASE_STEMS))[pi]
                if h > 0:
                    svg.rect(x, ty(acc), slot * 0.42, ty(acc + h) - ty(acc), PHASE_COLORS[stem])
                acc += h
        if len(order) <= 60:
            svg.text(LEFT + slot * (k + 0.5), H - BOTTOM + 12, str(idx))
    for i, stem in enumerate(PHASE_STEMS):  # legend, upper right
        y = TOP + 8 + 11 * i
        svg.rect(W - RIGHT - 110, y - 7, 9, 8, PHASE_COLORS[stem])
        svg.text(W - RIGHT - 97, y, stem, anchor="start", size=7)
    return svg.done()


def main(argv: list[str] | None = None) -> int:
    ap = argparse.ArgumentParser(prog="charts")
    sub = ap.add_subparsers(dest="kind", required=True)
    for kind in ("speedup", "breakdown"):
        p = sub.add_parser(kind)
        p.add_argument("--in", dest="input_path", required=True)
        p.add_argument("--out", dest="output_path", required=True)
        p.add_argument("--scope", default="convolution", choices=list(SCOPES))
        p.add_argument("--sort", default="convset-order", choices=list(SORTS))
        p.add_argument("--log-y", action="store_true")
    a = ap.parse_args(argv)
    try:
        out = (speedup_svg(a.input_path, a.scope, a.sort, a.log_y) if a.kind == "speedup"
               else breakdown_svg(a.input_path))
        with open(a.output_path, "w", encoding="utf-8") as fh:
            fh.write(out)
    except (OSError, ChartDataError) as exc:
        print(f"charts: {exc}", file=sys.stderr)
        return 1
    return 0


if __name__ == "__main__":
    sys.exit(main())
