"""The per-step timer (TM-Tool): same contract as the reference ledger (reference
tests/test_timing.py and test_acceptance.py:89-136), CPU only."""

from __future__ import annotations

import random

import pytest

from paper_2407_10730_b200.timing import (IN_PHASES, PHASE_COLUMNS, Phase, PhaseLedger,
                                          TimingStateError, aggregate)


def test_phase_nomenclature_matches_reference():
    assert [p.name for p in Phase] == ["PRE_ANALYSIS", "PRE_REORDER", "IN_TILING", "IN_PACKING",
                                       "IN_MICROKERNEL", "IN_UNPACKING", "POST_REORDER"]
    assert [int(p) for p in Phase] == list(range(7))
    assert IN_PHASES == (Phase.IN_TILING, Phase.IN_PACKING, Phase.IN_MICROKERNEL, Phase.IN_UNPACKING)
    assert PHASE_COLUMNS[Phase.IN_MICROKERNEL] == "in_microkernel"


def test_errors(fake_clock):
    led = PhaseLedger(clock=fake_clock)
    led.start(Phase.IN_PACKING)
    with pytest.raises(TimingStateError, match="already started"):
        led.start(Phase.IN_PACKING)
    with pytest.raises(TimingStateError, match="pending"):
        led.snapshot()
    with pytest.raises(TimingStateError, match="without a matching start"):
        led.update(Phase.POST_REORDER)


def test_independent_phases_and_accumulation(fake_clock):
    led = PhaseLedger(clock=fake_clock)
    led.start(Phase.IN_PACKING)
    fake_clock.advance(5)
    led.start(Phase.IN_MICROKERNEL)
    fake_clock.advance(7)
    led.update(Phase.IN_PACKING)
    led.update(Phase.IN_MICROKERNEL)
    for dt in (3, 11, 5):
        led.start(Phase.IN_TILING)
        fake_clock.advance(dt)
        led.update(Phase.IN_TILING)
    r = led.snapshot()
    assert r.elapsed_ns[Phase.IN_PACKING] == 12 and r.elapsed_ns[Phase.IN_MICROKERNEL] == 7
    assert r.calls[Phase.IN_TILING] == 3 and r.elapsed_ns[Phase.IN_TILING] == 19
    assert r.operation_ns == 38 and r.convolution_ns == 38
    led.reset()
    assert led.snapshot().operation_ns == 0


def test_aggregate_mean_min_and_divergence(fake_clock):
    reps = []
    for dt in (10, 30, 20):
        led = PhaseLedger(clock=fake_clock)
        led.start(Phase.PRE_REORDER)
        fake_clock.advance(dt)
        led.update(Phase.PRE_REORDER)
        reps.append(led.snapshot())
    st = aggregate(reps)
    assert st.runs == 3 and st.phase_ns_mean[Phase.PRE_REORDER] == 20
    assert st.phase_ns_min[Phase.PRE_REORDER] == 10 and st.operation_ns_min == 10
    led = PhaseLedger(clock=fake_clock)
    with pytest.raises(ValueError, match="diverge"):
        aggregate([reps[0], led.snapshot()])
    with pytest.raises(ValueError):
        aggregate([])


def test_random_balanced_interleavings(fake_clock):
    rng = random.Random(9)
    for _ in range(300):
        led = PhaseLedger(clock=fake_clock)
        open_at, el, calls = {}, {p: 0 for p in Phase}, {p: 0 for p in Phase}
        for _ in range(rng.randint(0, 40)):
            fake_clock.advance(rng.randint(0, 997))
            can = [p for p in Phase if p not in open_at]
            if open_at and (not can or rng.random() < 0.5):
                p = rng.choice(sorted(open_at))
                el[p] += fake_clock.t - open_at.pop(p)
                calls[p] += 1
                led.update(p)
            else:
                p = rng.choice(can)
                open_at[p] = fake_clock.t
                led.start(p)
        for p in sorted(open_at):
            el[p] += fake_clock.t - open_at[p]
            calls[p] += 1
            led.update(p)
        r = led.snapshot()
        assert dict(r.calls) == calls and dict(r.elapsed_ns) == el
        assert r.operation_ns == sum(el.values())
        assert r.convolution_ns == sum(el[p] for p in IN_PHASES)


def test_reference_ledger_interchangeable():
    """The GPU drop-ins accept the reference's own PhaseLedger: phase ids are the same
    IntEnum values, so a reference ledger indexes them identically."""
    led = PhaseLedger()
    led.start(3)
    led.update(Phase(3))
    assert led.snapshot().calls[Phase.IN_PACKING] == 1
