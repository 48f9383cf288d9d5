"""Results CSV in the reference schema (reference pkg/src/convbench/report.py:21-27,40-93).

One row per operation outcome: key, mode, status, runs, warmups; mean / min / calls of
every phase in Phase order; operation and convolution mean / min; correctness error.
Files written here are read unchanged by the reference's `convbench report`.
"""

from __future__ import annotations

import csv
from dataclasses import dataclass
from pathlib import Path

from .harness import RunOutcome
from .timing import PHASE_COLUMNS, Phase

RESULTS_HEADER = ["key", "mode", "status", "runs", "warmups"]
for _p in Phase:
    RESULTS_HEADER += [f"{PHASE_COLUMNS[_p]}_ns_mean", f"{PHASE_COLUMNS[_p]}_ns_min",
                       f"{PHASE_COLUMNS[_p]}_calls"]
RESULTS_HEADER += ["operation_ns_mean", "operation_ns_min", "convolution_ns_mean",
                   "convolution_ns_min", "correctness_max_rel_err"]


def _fmt(v) -> str:
    return "" if v is None else repr(float(v)) if isinstance(v, float) else str(v)


def outcome_record(o: RunOutcome) -> list[str]:
    rec = [o.key, o.mode, o.status, str(o.runs), str(o.warmups)]
    s = o.stats
    for p in Phase:
        rec += ["", "", ""] if s is None else [_fmt(float(s.phase_ns_mean[p])),
                                               _fmt(int(s.phase_ns_min[p])), _fmt(int(s.calls[p]))]
    if s is None:
        rec += ["", "", "", ""]
    else:
        rec += [_fmt(float(s.operation_ns_mean)), _fmt(int(s.operation_ns_min)),
                _fmt(float(s.convolution_ns_mean)), _fmt(int(s.convolution_ns_min))]
    rec.append(_fmt(o.correctness_max_rel_err))
    return rec


def write_results_csv(outcomes, path: str | Path) -> None:
    """Write outcomes (RunOutcome or pre-formatted records) in the reference schema."""
    outcomes = list(outcomes)
    if not outcomes:
        raise ValueError("refusing to write an empty results file")
    with open(path, "w", newline="", encoding="utf-8") as fh:
        w = csv.writer(fh)
        w.writerow(RESULTS_HEADER)
        for o in outcomes:
            w.writerow(o if isinstance(o, list) else outcome_record(o))


@dataclass
class ResultRow:
    key: str
    mode: str
    status: str
    operation_ns_mean: float | None
    operation_ns_min: int | None
    phase_ns_mean: dict


def read_results_csv(path: str | Path) -> list[ResultRow]:
    rows = []
    with open(path, newline="", encoding="utf-8") as fh:
        r = csv.reader(fh)
        header = next(r)
        if header != RESULTS_HEADER:
            raise ValueError(f"{path}: header does not match the results schema")
        for rec in r:
            d = dict(zip(header, rec))
            f = lambda k: float(d[k]) if d[k] != "" else None
            rows.append(ResultRow(
                key=d["key"], mode=d["mode"], status=d["status"],
                operation_ns_mean=f("operation_ns_mean"),
                operation_ns_min=int(d["operation_ns_min"]) if d["operation_ns_min"] else None,
                phase_ns_mean={p: f(f"{PHASE_COLUMNS[p]}_ns_mean") for p in Phase}))
    return rows
