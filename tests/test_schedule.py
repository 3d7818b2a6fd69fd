"""The B200 runner's schedule module vs the reference's timelines (CPU).

Golden fixtures: tests/golden/schedule_golden.json (made by the reference's
build_1f1b / update_gaps / bubble_ratio / makespan). Property tests follow
pkg/tests/test_schedule.py.
"""

import json
from fractions import Fraction
from pathlib import Path

import pytest

from paper_2312_00839_b200.errors import TimelineError
from paper_2312_00839_b200.schedule import (
    BACKWARD,
    FORWARD,
    TIMELINE_CSV_HEADER,
    UPDATE,
    CostModel,
    ScheduleEvent,
    Timeline,
    bubble_ratio,
    build_1f1b,
    build_gpipe,
    build_naive,
    build_serial,
    count_updates_between,
    makespan,
    stage_program,
    steady_state_window,
    timeline_csv_text,
    timeline_from_json_obj,
    timeline_json_obj,
    update_gaps,
    validate_timeline,
)

GOLDEN = json.loads((Path(__file__).resolve().parent / "golden" / "schedule_golden.json").read_text())


def test_1f1b_matches_reference_bit_exactly():
    """Per-stage event order, slots, global order, gaps, horizon, bubbles,
    steady window and makespan == the reference, D = 1..8."""
    for case in GOLDEN:
        D, n = case["depth"], case["n"]
        tl = build_1f1b(D, n)
        validate_timeline(tl)
        for k in range(D):
            evs = tl.stage_events(k)
            assert [f"{e.kind[0].upper()}{e.mb}" for e in evs] == case["stages"][k]["seq"]
            assert [e.slot for e in evs] == case["stages"][k]["slots"]
        assert [[e.slot, e.stage, e.kind[0].upper(), e.mb] for e in tl.events] == case["global"]
        assert sorted([mb, k, s] for (mb, k), s in update_gaps(tl).items()) == case["gaps"]
        assert tl.horizon == case["horizon"]
        assert str(bubble_ratio(tl)) == case["bubble"]
        steady = steady_state_window(tl)
        assert (list(steady) if steady else None) == case["steady"]
        if steady:
            assert str(bubble_ratio(tl, *steady)) == case["bubble_steady"]
        assert makespan(tl) == case["makespan"]


def test_warm_up_counts_and_gaps():
    depth = 4
    tl = build_1f1b(depth, 12)
    for k in range(depth):
        evs = tl.stage_events(k)
        first_b = next(i for i, e in enumerate(evs) if e.kind == BACKWARD)
        assert sum(1 for e in evs[:first_b] if e.kind == FORWARD) == depth - k
    for (mb, k), s in update_gaps(tl).items():
        assert s == min(mb - 1, depth - k - 1)


def test_worked_example_slots():
    slots = {(e.kind, e.mb): e.slot for e in build_1f1b(4, 8).stage_events(0)}
    assert slots[(FORWARD, 1)] == 0 and slots[(FORWARD, 4)] == 3
    assert slots[(BACKWARD, 1)] == 7 and slots[(FORWARD, 5)] == 8 and slots[(BACKWARD, 5)] == 15


@pytest.mark.parametrize("depth", [2, 3, 4, 8])
def test_steady_gap_equals_version_difference(depth):
    n = depth + 20
    tl = build_1f1b(depth, n)
    for k in range(depth):
        for m in range(depth, n + 1):
            assert count_updates_between(tl, k, (FORWARD, m), (BACKWARD, m)) == depth - k - 1


def test_count_updates_between_errors():
    tl = build_1f1b(2, 4)
    with pytest.raises(TimelineError):
        count_updates_between(tl, 0, (FORWARD, 99), (BACKWARD, 1))
    with pytest.raises(TimelineError):
        count_updates_between(tl, 0, (BACKWARD, 3), (FORWARD, 3))


def test_makespans_and_bubbles():
    depth, n = 4, 16
    assert makespan(build_1f1b(depth, n)) == 2 * n + 2 * depth - 2
    assert makespan(build_naive(depth, n)) == 2 * depth * n
    assert makespan(build_1f1b(depth, n)) <= makespan(build_gpipe(depth, n, 4)) <= makespan(build_naive(depth, n))
    assert makespan(build_serial(4), CostModel([3.0], [2.0])) == 20
    tl = build_1f1b(4, 10)
    assert makespan(tl, CostModel(2.0, 2.0)) == 2 * makespan(tl)
    assert bubble_ratio(build_naive(4, 6)) == Fraction(3, 4)
    assert bubble_ratio(build_gpipe(4, 1, 4)) == Fraction(3, 7)
    tl = build_1f1b(4, 20)
    start, end = steady_state_window(tl)
    assert start == 7 and end - start >= 10 and bubble_ratio(tl, start, end) == 0
    with pytest.raises(TimelineError):
        bubble_ratio(build_serial(2), 3, 3)


def test_depth_one_is_serial():
    key = lambda tl: {(e.slot, e.stage, e.kind, e.mb, e.micro) for e in tl.events}  # noqa: E731
    assert key(build_1f1b(1, 9)) == key(build_serial(9))
    assert key(build_naive(1, 7)) == key(build_serial(7))
    assert key(build_gpipe(4, 5, 1)) == key(build_naive(4, 5))


@pytest.mark.parametrize("depth", list(range(1, 9)))
@pytest.mark.parametrize("n", [1, 2, 3, 8, 32])
def test_validator_accepts_builders(depth, n):
    validate_timeline(build_naive(depth, n))
    validate_timeline(build_1f1b(depth, n))
    for t in (1, 2, 4):
        validate_timeline(build_gpipe(depth, n, t))


def test_validator_rejects_corruption():
    tl = build_1f1b(3, 4)
    bad, moved = [], False
    for e in tl.events:
        if not moved and e.kind == BACKWARD and e.mb == 2 and e.stage == 0:
            bad.append(ScheduleEvent(0, e.stage, e.kind, e.mb, e.micro))
            moved = True
        else:
            bad.append(e)
    with pytest.raises(TimelineError):
        validate_timeline(Timeline(tl.kind, tl.depth, tl.n_batches, 1, bad))
    ev = [ScheduleEvent(0, 0, FORWARD, 1), ScheduleEvent(0, 0, BACKWARD, 1), ScheduleEvent(0, 0, UPDATE, 1)]
    with pytest.raises(TimelineError):
        validate_timeline(Timeline("serial", 1, 1, 1, ev))


def test_export_round_trip():
    text = timeline_csv_text(build_serial(1)).strip().split("\n")
    assert text[0] == TIMELINE_CSV_HEADER == "slot,stage,kind,mb,micro"
    assert text[1] == "0,0,forward,1,0" and len(text) == 4
    tl = build_gpipe(3, 2, 2)
    back = timeline_from_json_obj(timeline_json_obj(tl))
    assert back.events == tl.events


@pytest.mark.parametrize("depth", [1, 2, 4, 8])
def test_stage_program_fusion_marks(depth):
    """Every update on a non-last stage that is immediately followed by a
    forward is marked for K3, with that forward's mb and gap; all
    steady-state updates qualify."""
    n = 3 * depth + 2
    tl = build_1f1b(depth, n)
    gaps = update_gaps(tl)
    for k in range(depth):
        prog = stage_program(tl, k)
        assert [(o.kind, o.mb) for o in prog] == [(e.kind, e.mb) for e in tl.stage_events(k)]
        fused = [o for o in prog if o.fuse_predict]
        if k == depth - 1:
            assert not fused
            assert all(o.gap is None for o in prog)
            continue
        for i, o in enumerate(prog):
            if o.kind == FORWARD:
                assert o.gap == gaps[(o.mb, k)]
            if o.kind == UPDATE:
                follows_fwd = i + 1 < len(prog) and prog[i + 1].kind == FORWARD
                assert o.fuse_predict == follows_fwd
                if follows_fwd:
                    assert (o.next_mb, o.next_gap) == (prog[i + 1].mb, prog[i + 1].gap)
        # updates not fused are exactly the drain: the last D-k-1 updates ... plus none in steady state
        assert len(fused) == n - (depth - k)
    live = stage_program(tl, 0, predictive=False)
    assert not any(o.fuse_predict for o in live)


def test_execute_rejects_unknown_stream_mode():
    import pytest

    from paper_2312_00839_b200.runtime import build_timeline, execute

    tl = build_timeline("async_raw", 2, 4)
    with pytest.raises(ValueError, match="streams"):
        execute(tl, [None, None], [None, None], "async_raw", None, "mse", lambda mb: 0.1, streams="bogus")
