"""Per-step (phase) timing: the TM-Tool nomenclature of the paper, host and CUDA-event clocks.

Mirrors convbench.timing (reference pkg/src/convbench/timing.py):
* Phase / IN_PHASES / PHASE_COLUMNS   timing.py:28-49
* TimingStateError, TimingReport       timing.py:52-62
* PhaseLedger (host monotonic ns)      timing.py:65-108, same start/update/reset/snapshot
                                       contract and the same errors
* RunStats / aggregate                 timing.py:111-151

and adds EventLedger, the GPU per-step timer: every device phase is a
pair of CUDA events recorded on the launching stream, resolved to integer nanoseconds
(round(ms * 1e6)) only at snapshot(), so timing never synchronises the pipeline.  Host
phases (operation analysis and tiling, which are host-side planning in the GPU
algorithms) keep the monotonic host clock.
"""

from __future__ import annotations

import enum
import time
from dataclasses import dataclass
from typing import Callable, Iterable, Mapping, Sequence


class Phase(enum.IntEnum):
    PRE_ANALYSIS = 0
    PRE_REORDER = 1
    IN_TILING = 2
    IN_PACKING = 3
    IN_MICROKERNEL = 4
    IN_UNPACKING = 5
    POST_REORDER = 6


IN_PHASES = (Phase.IN_TILING, Phase.IN_PACKING, Phase.IN_MICROKERNEL, Phase.IN_UNPACKING)

PHASE_COLUMNS = {p: p.name.lower() for p in Phase}

HOST_PHASES = frozenset({Phase.PRE_ANALYSIS, Phase.IN_TILING})


class TimingStateError(RuntimeError):
    """Unbalanced or misplaced start/update calls."""


@dataclass(frozen=True)
class TimingReport:
    elapsed_ns: Mapping[Phase, int]
    calls: Mapping[Phase, int]
    operation_ns: int
    convolution_ns: int


def _report(elapsed: Sequence[int], calls: Sequence[int]) -> TimingReport:
    return TimingReport(
        elapsed_ns={p: int(elapsed[p]) for p in Phase},
        calls={p: int(calls[p]) for p in Phase},
        operation_ns=int(sum(elapsed)),
        convolution_ns=int(sum(elapsed[p] for p in IN_PHASES)),
    )


class PhaseLedger:
    """Integer-ns accumulator per phase with call counts; the clock is injectable."""

    device_timed = False

    def __init__(self, clock: Callable[[], int] = time.perf_counter_ns) -> None:
        self._clock = clock
        self.reset()

    def reset(self) -> None:
        n = len(Phase)
        self._elapsed = [0] * n
        self._calls = [0] * n
        self._pending: list[int | None] = [None] * n

    def start(self, phase: Phase) -> None:
        if self._pending[phase] is not None:
            raise TimingStateError(f"start({Phase(phase).name}) while already started")
        self._pending[phase] = self._clock()

    def update(self, phase: Phase) -> None:
        t0 = self._pending[phase]
        if t0 is None:
            raise TimingStateError(f"update({Phase(phase).name}) without a matching start")
        self._elapsed[phase] += self._clock() - t0
        self._calls[phase] += 1
        self._pending[phase] = None

    def _check_balanced(self) -> None:
        open_ = [p.name for p in Phase if self._pending[p] is not None]
        if open_:
            raise TimingStateError(f"snapshot with pending starts: {', '.join(open_)}")

    def snapshot(self) -> TimingReport:
        self._check_balanced()
        return _report(self._elapsed, self._calls)


class EventLedger(PhaseLedger):
    """PhaseLedger whose device phases are timed with CUDA events on `stream`.

    start/update only *record* events (asynchronous; raw events through the C ABI,
    cb_event_record, about 1 us of host time each); snapshot() waits for the last event
    and converts every pair to integer ns.  Phases in `host_phases` use the host clock
    exactly like PhaseLedger.  Without an explicit `stream`, events go to the stream that
    is current at the first record of a run (after reset()); external ledgers resolve it
    at every record, since they are recorded inside graph captures.
    """

    device_timed = True

    def __init__(self, stream=None, host_phases: Iterable[Phase] = HOST_PHASES,
                 clock: Callable[[], int] = time.perf_counter_ns, external: bool = False) -> None:
        import torch  # plumbing only: the current stream
        from . import _capi

        self._torch = torch
        self._capi = _capi
        self._lib = _capi.load()
        self._stream = stream
        self._host = frozenset(Phase(p) for p in host_phases)
        # external events may be recorded inside a CUDA-graph capture: the graph then
        # re-records them on every replay, so snapshot() reads the latest replay's times
        self._external = 1 if external else 0
        self._pool: list[int] = []
        self._st = None
        super().__init__(clock)

    def reset(self) -> None:
        super().reset()
        pool = getattr(self, "_pool", [])
        for pair in getattr(self, "_pairs", []):
            pool.extend(pair[1:])
        self._pool = pool
        self._pairs: list[tuple[Phase, int, int]] = []
        self._open_evt: list[int | None] = [None] * len(Phase)
        self._st = None

    def __del__(self) -> None:
        lib = getattr(self, "_lib", None)
        if lib is None:
            return
        evs = list(getattr(self, "_pool", []))
        for pair in getattr(self, "_pairs", []):
            evs.extend(pair[1:])
        for e in evs:
            try:
                lib.cb_event_destroy(e)
            except Exception:  # interpreter shutdown
                pass

    def _event(self) -> int:
        if self._pool:
            return self._pool.pop()
        import ctypes
        h = ctypes.c_void_p()
        self._capi.check(self._lib.cb_event_create(ctypes.byref(h)))
        return h.value

    def _stream_handle(self) -> int:
        if self._st is None or self._external:
            s = self._stream if self._stream is not None else self._torch.cuda.current_stream()
            st = getattr(s, "cuda_stream", s)
            if self._external:
                return st
            self._st = st
        return self._st

    def _record(self) -> int:
        ev = self._event()
        self._capi.check(self._lib.cb_event_record(ev, self._stream_handle(), self._external))
        return ev

    def start(self, phase: Phase) -> None:
        phase = Phase(phase)
        if phase in self._host:
            return super().start(phase)
        if self._open_evt[phase] is not None:
            raise TimingStateError(f"start({phase.name}) while already started")
        self._open_evt[phase] = self._record()

    def update(self, phase: Phase) -> None:
        phase = Phase(phase)
        if phase in self._host:
            return super().update(phase)
        ev0 = self._open_evt[phase]
        if ev0 is None:
            raise TimingStateError(f"update({phase.name}) without a matching start")
        ev1 = self._record()
        self._pairs.append((phase, ev0, ev1))
        self._open_evt[phase] = None

    def snapshot(self) -> TimingReport:
        import ctypes
        open_ = [p.name for p in Phase
                 if self._pending[p] is not None or self._open_evt[p] is not None]
        if open_:
            raise TimingStateError(f"snapshot with pending starts: {', '.join(open_)}")
        elapsed = list(self._elapsed)
        calls = list(self._calls)
        ns = ctypes.c_int64()
        for phase, e0, e1 in self._pairs:
            self._capi.check(self._lib.cb_event_elapsed_ns(e0, e1, ctypes.byref(ns)))
            elapsed[phase] += ns.value
            calls[phase] += 1
        return _report(elapsed, calls)


@dataclass(frozen=True)
class RunStats:
    runs: int
    phase_ns_mean: Mapping[Phase, float]
    phase_ns_min: Mapping[Phase, int]
    calls: Mapping[Phase, int]
    operation_ns_mean: float
    operation_ns_min: int
    convolution_ns_mean: float
    convolution_ns_min: int


def aggregate(reports: Sequence[TimingReport]) -> RunStats:
    """Mean/min per phase; call counts must agree across runs (timing.py:130-151)."""
    if not reports:
        raise ValueError("aggregate() needs at least one report")
    calls0 = dict(reports[0].calls)
    for i, r in enumerate(reports[1:], start=1):
        if dict(r.calls) != calls0:
            raise ValueError(f"call counts diverge between run 0 and run {i}: "
                             f"{calls0} vs {dict(r.calls)}")
    n = len(reports)
    mean = {p: sum(r.elapsed_ns[p] for r in reports) / n for p in Phase}
    mins = {p: min(r.elapsed_ns[p] for r in reports) for p in Phase}
    return RunStats(
        runs=n,
        phase_ns_mean=mean,
        phase_ns_min=mins,
        calls=calls0,
        operation_ns_mean=sum(r.operation_ns for r in reports) / n,
        operation_ns_min=sum(mins.values()),
        convolution_ns_mean=sum(r.convolution_ns for r in reports) / n,
        convolution_ns_min=sum(mins[p] for p in IN_PHASES),
    )
