"""Config-5 sweep with CPU-oracle parity on every op -- TEST INFRASTRUCTURE (not collected).

    python tests/sweep_parity.py --out sweep_out [--gpus N] [--sample K] [sweep.py options]

Runs tools/sweep.py (timing every op in every mode on make_inputs data through the package
harness) and hands each op's outputs to the oracle checker below: a pool of host worker
processes regenerates the op's inputs (oracle/conv_oracle.make_inputs, bit-identical),
computes the float64 reference (oracle.conv_banded64 -- conv_direct_naive's sums in
another order, algos.py:212-240) and reports

    err = max|y_gpu - y_ref| / sqrt(C/g * R * S)       (gate: <= 1e-4, BASELINE.json)

plus the reference allclose's max_rel_err (tensor.py:46-65, informational).  Duplicate ops
share one oracle computation (make_inputs seeds from the op key) but every occurrence's
output is checked.  GPU outputs travel to the workers as .npy files in a RAM-backed
directory; at most --pending keys are in flight, so memory stays bounded while the GPU
keeps running.

Outputs (rank 0): sweep.py's results CSVs and summary.json, with a "parity" block per
mode (checked / unchecked counts, max / p99 / p50 error, the worst op, ops over the
gate), and parity.csv (one row per op and mode).
"""

from __future__ import annotations

import csv
import importlib.util
import math
import os
import platform
import shutil
import sys
import tempfile
import time
from concurrent.futures import ProcessPoolExecutor
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

import numpy as np

TOL = 1e-4


def _sweep_module():
    spec = importlib.util.spec_from_file_location("sweep_tool", ROOT / "tools" / "sweep.py")
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def _worker_init(root: str) -> None:
    if root not in sys.path:
        sys.path.insert(0, root)
    from threadpoolctl import threadpool_limits
    threadpool_limits(1)  # one core per worker: the pool is the parallelism


def oracle_channels(desc, max_flops: float) -> np.ndarray | None:
    """Output channels the oracle computes for one op: all of them (None) up to max_flops of
    oracle work, else a seeded subset of ceil(K * max_flops / flops) >= 8 channels (every
    pixel of each), so the sweep's largest ops (up to 2e13 FLOPs) are checked too."""
    from paper_2407_10730_b200.descriptor import flop_count, key_of
    f = flop_count(desc)
    if f <= max_flops or desc.groups != 1:
        return None
    k = min(desc.out_channels, max(8, math.ceil(desc.out_channels * max_flops / f)))
    rng = np.random.default_rng(int.from_bytes(key_of(desc).encode()[-8:], "little"))
    return np.sort(rng.choice(desc.out_channels, size=k, replace=False))


def _check_job(desc, data_seed: int, items: list, channels=None) -> list:
    """Oracle of one op key (all output channels, or `channels`), compared with every output
    of that key."""
    from dataclasses import replace
    from oracle import conv_oracle as orc
    t0 = time.perf_counter()
    x, w, b = orc.make_inputs(desc, data_seed)
    if channels is not None:  # the same conv restricted to a subset of output channels
        d_sub = replace(desc, out_channels=len(channels))
        ref64 = orc.conv_banded64(d_sub, x, np.ascontiguousarray(w[channels]),
                                  None if b is None else b[channels])
    else:
        ref64 = orc.conv_banded64(desc, x, w, b)
    want = ref64.astype(np.float32)  # conv_direct_naive's output: one final fp32 rounding
    red = orc.reduction_len(desc)
    t_ref = time.perf_counter() - t0
    note0 = None if channels is None else f"{len(channels)}/{desc.out_channels} channels"
    res = []
    for index, mode, path in items:
        y = np.load(path, mmap_mode="r")
        if channels is not None and y.ndim == 4:
            y = y[:, channels]
        y = np.ascontiguousarray(y)
        os.unlink(path)
        if y.shape != want.shape:
            res.append((index, mode, math.inf, math.inf, f"shape {y.shape} != {want.shape}"))
            continue
        err = orc.normalized_max_err(y, want, red)
        rel = orc.reference_allclose_err(y, want)
        res.append((index, mode, err, rel, note0))
    return [(i, m, e, r, note, t_ref) for i, m, e, r, note in res]


class OracleChecker:
    def __init__(self, data_seed: int, workers: int, pending: int, spool: str | None = None,
                 journal: str | None = None, max_oracle_flops: float = 3e10):
        import multiprocessing as mp
        self.max_oracle_flops = max_oracle_flops
        self.journal = open(journal, "a") if journal else None  # results as they arrive
        self.data_seed = data_seed
        self.workers = workers
        self.pending_max = pending
        base = spool or ("/dev/shm" if os.path.isdir("/dev/shm") else None)
        self.dir = tempfile.mkdtemp(prefix="cb_parity_", dir=base)
        self.pool = ProcessPoolExecutor(workers, mp_context=mp.get_context("spawn"),
                                        initializer=_worker_init, initargs=(str(ROOT),))
        self.futures = []
        self.results: dict[str, dict] = {}
        self.oracle_s = 0.0
        self.blocked_s = 0.0
        self.keys = 0

    def progress(self) -> str:
        return (f"(oracle: {len(self.results)} outputs checked, {len(self.futures)} keys pending, "
                f"{self.blocked_s:.0f} s blocked on the pool)")

    def _drain(self, keep: int) -> None:
        t0 = time.perf_counter()
        while len(self.futures) > keep:
            f = self.futures.pop(0)
            for i, m, e, r, note, t_ref in f.result():
                self.results[f"{i}:{m}"] = {"err": e, "allclose_rel_err": r, "note": note}
                if self.journal:
                    self.journal.write(f"{i},{m},{e:.4e},{r:.4e},{note or ''}\n")
            if self.journal:
                self.journal.flush()
            self.oracle_s += t_ref
        self.blocked_s += time.perf_counter() - t0

    def check(self, desc, host, outs) -> None:
        items = []
        for i, m, y in outs:
            path = os.path.join(self.dir, f"{i}_{m}.npy")
            np.save(path, y.cpu().numpy() if hasattr(y, "cpu") else np.asarray(y))
            items.append((i, m, path))
        if not items:
            return
        self.futures.append(self.pool.submit(_check_job, desc, self.data_seed, items,
                                             oracle_channels(desc, self.max_oracle_flops)))
        self.keys += 1
        self._drain(self.pending_max)

    def finish(self) -> dict:
        self._drain(0)
        self.pool.shutdown()
        shutil.rmtree(self.dir, ignore_errors=True)
        return self.results

    def summarize(self, mode: str, rows: list, parity: dict) -> dict:
        errs, unchecked, over = [], [], []
        for index, key, status in rows:
            r = parity.get(f"{index}:{mode}")
            if r is None:
                unchecked.append((index, key, status))
                continue
            errs.append((r["err"], index, key))
            if not r["err"] <= TOL:
                over.append((index, key, r["err"]))
        e = np.array([x[0] for x in errs], dtype=np.float64)
        worst = max(errs) if errs else None
        return {"gate": f"max|y - y_ref| / sqrt(C/g*R*S) <= {TOL:g}",
                "checked": len(errs), "unchecked": len(unchecked),
                "unchecked_ops": unchecked[:50],
                "over_gate": len(over), "over_gate_ops": over[:50],
                "max_err": float(e.max()) if e.size else None,
                "p99_err": float(np.percentile(e, 99)) if e.size else None,
                "p50_err": float(np.percentile(e, 50)) if e.size else None,
                "worst_op": {"index": worst[1], "key": worst[2], "err": worst[0]} if worst else None,
                "max_allclose_rel_err": max((parity[f"{i}:{mode}"]["allclose_rel_err"]
                                             for i, _, _ in rows if f"{i}:{mode}" in parity),
                                            default=None)}

    def describe(self) -> dict:
        cpu = platform.processor() or ""
        try:
            with open("/proc/cpuinfo") as f:
                cpu = next((ln.split(":", 1)[1].strip() for ln in f if ln.startswith("model name")), cpu)
        except OSError:
            pass
        return {"oracle": "oracle/conv_oracle.conv_banded64 (float64 im2col GEMM over row bands; "
                          "conv_direct_naive's sums, algos.py:212-240), rounded once to fp32",
                "inputs": "oracle/conv_oracle.make_inputs (bit-identical to harness.py:79-96)",
                "workers_per_rank": self.workers, "host_cpu": cpu, "cpu_count": os.cpu_count(),
                "coverage": f"every output of ops up to {self.max_oracle_flops / 1e9:g} GFLOP; "
                            "larger ops: every pixel of a seeded subset of ceil(K * limit / "
                            "flops) >= 8 output channels (note column of parity.csv)",
                "oracle_cpu_s": self.oracle_s, "unique_keys_checked": self.keys}

    @staticmethod
    def write_table(path: Path, descs, parity: dict) -> None:
        from paper_2407_10730_b200.descriptor import key_of
        rows = sorted(((int(k.split(":")[0]), k.split(":")[1], v) for k, v in parity.items()),
                      key=lambda r: (r[0], r[1]))
        with open(path, "w", newline="") as f:
            wr = csv.writer(f)
            wr.writerow(["index", "key", "mode", "normalized_max_err", "allclose_rel_err", "note"])
            for i, m, v in rows:
                wr.writerow([i, key_of(descs[i]), m, f"{v['err']:.4e}",
                             f"{v['allclose_rel_err']:.4e}", v["note"] or ""])


def main(argv=None) -> int:
    argv = sys.argv[1:] if argv is None else list(argv)
    extra = {"--workers": 0, "--pending": 24, "--max-oracle-gflop": 30}
    rest = []
    it = iter(argv)
    for a in it:
        if a in extra:
            extra[a] = float(next(it)) if a == "--max-oracle-gflop" else int(next(it))
        else:
            rest.append(a)
    sweep = _sweep_module()

    def factory(args, ranks):
        # leave cores for the ranks' own host work (input generation, D2H, spooling)
        workers = extra["--workers"] or max(1, (os.cpu_count() or 2) // ranks.world - 2)
        os.makedirs(args.out, exist_ok=True)
        return OracleChecker(args.data_seed, workers, extra["--pending"],
                             journal=os.path.join(args.out, f"parity_rank{ranks.rank}.journal.csv"),
                             max_oracle_flops=extra["--max-oracle-gflop"] * 1e9)
    return sweep.main(rest, checker_factory=factory, script=str(Path(__file__).resolve()),
                      relaunch_argv=argv)


if __name__ == "__main__":
    sys.exit(main())
