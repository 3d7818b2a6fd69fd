"""Slot timelines for the pipeline schedules and the per-stage programs the
B200 runner executes.

Mirrors the reference's schedule API (pkg/src/pipesim/schedule.py): event
kinds, `ScheduleEvent`, `Timeline` (global order = (slot, stage, kind) with an
UPDATE after the same-slot BACKWARD, schedule.py:28,74), the builders, the
validator and the analyses. The 1F1B builder is the hot-path one
(schedule.py:150-172); serial / naive / GPipe are provided for the same
Timeline API.

What the B200 runtime consumes is `stage_program(tl, k)`: stage k's events in
execution order, each annotated with what the stage needs to know locally —
the peer it receives from / sends to and, for predictive forwards, the
timeline-exact version gap `s` (runtime.py:300-315) — so every rank can run
its program without consulting the global timeline.
"""

from __future__ import annotations

import json
from dataclasses import dataclass, field
from fractions import Fraction

from .errors import TimelineError

FORWARD = "forward"
BACKWARD = "backward"
UPDATE = "update"

# forward/backward occupy the slot; an update shares its backward's slot and
# sorts after it (schedule.py:28)
_KIND_RANK = {FORWARD: 0, BACKWARD: 0, UPDATE: 1}

TIMELINE_CSV_HEADER = "slot,stage,kind,mb,micro"


@dataclass(frozen=True)
class ScheduleEvent:
    slot: int
    stage: int
    kind: str
    mb: int
    micro: int = 0


@dataclass
class CostModel:
    """Per-stage forward/backward durations (scalars or per-stage lists);
    updates are free; micro-batched events scale by 1/micro_per_mini
    (schedule.py:44-62)."""

    forward_cost: float | list[float] = 1.0
    backward_cost: float | list[float] = 1.0

    @staticmethod
    def _pick(c, stage):
        return float(c[stage]) if isinstance(c, (list, tuple)) else float(c)

    def fcost(self, stage: int) -> float:
        return self._pick(self.forward_cost, stage)

    def bcost(self, stage: int) -> float:
        return self._pick(self.backward_cost, stage)


def _order_key(e: ScheduleEvent):
    return (e.slot, e.stage, _KIND_RANK[e.kind])


@dataclass
class Timeline:
    kind: str
    depth: int
    n_batches: int
    micro_per_mini: int
    events: list[ScheduleEvent] = field(default_factory=list)

    def __post_init__(self):
        self.events = sorted(self.events, key=_order_key)

    @property
    def horizon(self) -> int:
        return 1 + max((e.slot for e in self.events), default=-1)

    def stage_events(self, stage: int) -> list[ScheduleEvent]:
        return [e for e in self.events if e.stage == stage]


def _check_depth(depth: int) -> None:
    if depth < 1:
        raise TimelineError(f"depth must be >= 1, got {depth}")


def _check_batches(n: int) -> None:
    if n < 1:
        raise TimelineError(f"n_batches must be >= 1, got {n}")


# ---- builders ---------------------------------------------------------------------


def build_1f1b(depth: int, n_batches: int) -> Timeline:
    """One-forward-one-backward with per-backward updates (schedule.py:150-172).

    Closed form, stage k, mini-batch m (1-indexed), w = depth - k warm-up
    forwards:  forward slot  k + m - 1                 if m <= w
                             2*depth - k + 2*(m - w - 1) otherwise
               backward slot = update slot = 2*depth - 1 - k + 2*(m - 1)
    """
    _check_depth(depth)
    _check_batches(n_batches)
    events = []
    for k in range(depth):
        warm = depth - k
        for m in range(1, n_batches + 1):
            f = k + m - 1 if m <= warm else 2 * depth - k + 2 * (m - warm - 1)
            b = 2 * depth - 1 - k + 2 * (m - 1)
            events += [
                ScheduleEvent(f, k, FORWARD, m),
                ScheduleEvent(b, k, BACKWARD, m),
                ScheduleEvent(b, k, UPDATE, m),
            ]
    return Timeline("1f1b", depth, n_batches, 1, events)


def build_serial(n_batches: int) -> Timeline:
    """Depth 1: F at 2(m-1), B and U at 2m-1 (schedule.py:87-95)."""
    _check_batches(n_batches)
    events = []
    for m in range(1, n_batches + 1):
        events += [
            ScheduleEvent(2 * m - 2, 0, FORWARD, m),
            ScheduleEvent(2 * m - 1, 0, BACKWARD, m),
            ScheduleEvent(2 * m - 1, 0, UPDATE, m),
        ]
    return Timeline("serial", 1, n_batches, 1, events)


def build_naive(depth: int, n_batches: int) -> Timeline:
    """One mini-batch in flight (schedule.py:98-111)."""
    _check_depth(depth)
    _check_batches(n_batches)
    events = []
    for m in range(1, n_batches + 1):
        base = 2 * depth * (m - 1)
        for k in range(depth):
            back = base + 2 * depth - 1 - k
            events += [
                ScheduleEvent(base + k, k, FORWARD, m),
                ScheduleEvent(back, k, BACKWARD, m),
                ScheduleEvent(back, k, UPDATE, m),
            ]
    return Timeline("naive", depth, n_batches, 1, events)


def build_gpipe(depth: int, n_batches: int, micro_per_mini: int) -> Timeline:
    """Micro-batched fill/drain with a synchronous flush (schedule.py:114-147)."""
    _check_depth(depth)
    _check_batches(n_batches)
    if micro_per_mini < 1:
        raise TimelineError(f"micro_per_mini must be >= 1, got {micro_per_mini}")
    t = micro_per_mini
    span = t + depth - 1
    events = []
    for m in range(1, n_batches + 1):
        base = 2 * span * (m - 1)
        for k in range(depth):
            for mu in range(t):
                events.append(ScheduleEvent(base + mu + k, k, FORWARD, m, mu))
                events.append(
                    ScheduleEvent(base + span + (t - 1 - mu) + (depth - 1 - k), k, BACKWARD, m, mu)
                )
            events.append(ScheduleEvent(base + span + (t - 1) + (depth - 1 - k), k, UPDATE, m))
    return Timeline("gpipe", depth, n_batches, t, events)


# ---- validation -----------------------------------------------------------------------


def validate_timeline(tl: Timeline) -> None:
    """Structural invariants (schedule.py:188-268): fields in range, one work
    event per stage-slot, forward chain down / backward chain up, backward
    after its forward, one update per (mb, stage) in the slot of its last
    backward, work conserved per stage. Raises TimelineError on the first breach.
    """
    T = tl.micro_per_mini
    fwd, bwd, upd = {}, {}, {}
    occupied = set()
    for e in tl.events:
        if e.slot < 0:
            raise TimelineError(f"negative slot in {e}")
        if not 0 <= e.stage < tl.depth:
            raise TimelineError(f"stage out of range in {e}")
        if not 1 <= e.mb <= tl.n_batches:
            raise TimelineError(f"mb out of range in {e}")
        if not 0 <= e.micro < T:
            raise TimelineError(f"micro out of range in {e}")
        if e.kind == UPDATE:
            key = (e.mb, e.stage)
            if key in upd:
                raise TimelineError(f"duplicate update for mb {e.mb} stage {e.stage}")
            upd[key] = e.slot
            continue
        if e.kind not in (FORWARD, BACKWARD):
            raise TimelineError(f"unknown kind in {e}")
        cell = (e.stage, e.slot)
        if cell in occupied:
            raise TimelineError(f"two work events on stage {e.stage} slot {e.slot}")
        occupied.add(cell)
        table = fwd if e.kind == FORWARD else bwd
        key = (e.mb, e.micro, e.stage)
        if key in table:
            raise TimelineError(f"duplicate {e.kind} for mb/micro/stage {key}")
        table[key] = e.slot

    last = tl.depth - 1
    for m in range(1, tl.n_batches + 1):
        for mu in range(T):
            for k in range(tl.depth):
                key = (m, mu, k)
                if key not in fwd or key not in bwd:
                    raise TimelineError(f"missing forward/backward for {key}")
                if k > 0 and fwd[key] <= fwd[(m, mu, k - 1)]:
                    raise TimelineError(
                        f"forward of mb {m} micro {mu} at stage {k} does not follow stage {k - 1}"
                    )
                if k < last and bwd[key] <= bwd[(m, mu, k + 1)]:
                    raise TimelineError(
                        f"backward of mb {m} micro {mu} at stage {k} does not follow stage {k + 1}"
                    )
                if bwd[key] <= fwd[key]:
                    raise TimelineError(
                        f"backward of mb {m} micro {mu} at stage {k} does not follow its forward"
                    )
        for k in range(tl.depth):
            if (m, k) not in upd:
                raise TimelineError(f"missing update for mb {m} stage {k}")
            if upd[(m, k)] != max(bwd[(m, mu, k)] for mu in range(T)):
                raise TimelineError(
                    f"update for mb {m} stage {k} not in the slot of its last backward"
                )

    want = tl.n_batches * T
    for k in range(tl.depth):
        nf = sum(1 for key in fwd if key[2] == k)
        nb = sum(1 for key in bwd if key[2] == k)
        nu = sum(1 for key in upd if key[1] == k)
        if (nf, nb, nu) != (want, want, tl.n_batches):
            raise TimelineError(
                f"work not conserved on stage {k}: {nf} forwards, {nb} backwards, {nu} updates"
            )


# ---- version-gap bookkeeping -----------------------------------------------------------


def update_gaps(tl: Timeline) -> dict[tuple[int, int], int]:
    """Updates a stage applies strictly between each mini-batch's (micro 0)
    forward and backward there, keyed (mb, stage) — the timeline-exact
    prediction step count s (runtime.py:300-315). Under 1F1B this is
    min(mb - 1, depth - stage - 1): warm-up mini-batches get smaller s (S1).
    """
    gaps: dict[tuple[int, int], int] = {}
    for k in range(tl.depth):
        count = 0
        started: dict[int, int] = {}
        for e in tl.stage_events(k):
            if e.kind == UPDATE:
                count += 1
            elif e.micro == 0:
                if e.kind == FORWARD:
                    started[e.mb] = count
                else:
                    gaps[(e.mb, k)] = count - started[e.mb]
    return gaps


def count_updates_between(tl: Timeline, stage: int, from_event: tuple, to_event: tuple) -> int:
    """Updates on `stage` strictly between two of its events, selected as
    (kind, mb) or (kind, mb, micro) (schedule.py:322-353)."""

    def find(spec):
        kind, mb = spec[0], spec[1]
        micro = spec[2] if len(spec) > 2 else 0
        for e in tl.events:
            if e.stage == stage and e.kind == kind and e.mb == mb and e.micro == micro:
                return e
        raise TimelineError(f"no event {spec} on stage {stage}")

    a, b = find(from_event), find(to_event)
    ka, kb = (a.slot, _KIND_RANK[a.kind]), (b.slot, _KIND_RANK[b.kind])
    if kb < ka:
        raise TimelineError("to_event precedes from_event")
    return sum(
        1
        for e in tl.events
        if e.stage == stage and e.kind == UPDATE and ka < (e.slot, _KIND_RANK[e.kind]) < kb
    )


# ---- analyses ----------------------------------------------------------------------------


def bubble_ratio(tl: Timeline, start: int | None = None, end: int | None = None) -> Fraction:
    """Idle stage-slots / (depth x window), exact (schedule.py:274-290)."""
    lo = 0 if start is None else start
    hi = tl.horizon if end is None else end
    if hi <= lo:
        raise TimelineError(f"empty slot window [{lo}, {hi})")
    busy = {(e.stage, e.slot) for e in tl.events if e.kind != UPDATE and lo <= e.slot < hi}
    cells = tl.depth * (hi - lo)
    return Fraction(cells - len(busy), cells)


def steady_state_window(tl: Timeline) -> tuple[int, int] | None:
    """Longest half-open run of slots where every stage works (schedule.py:293-315)."""
    per_slot: dict[int, set[int]] = {}
    for e in tl.events:
        if e.kind != UPDATE:
            per_slot.setdefault(e.slot, set()).add(e.stage)
    full = sorted(s for s, st in per_slot.items() if len(st) == tl.depth)
    if not full:
        return None
    best_lo, best_hi = full[0], full[0]
    run_lo = run_hi = full[0]
    for s in full[1:] + [None]:
        if s is not None and s == run_hi + 1:
            run_hi = s
            continue
        if run_hi - run_lo > best_hi - best_lo:
            best_lo, best_hi = run_lo, run_hi
        if s is not None:
            run_lo = run_hi = s
    return best_lo, best_hi + 1


def makespan(tl: Timeline, costs: CostModel | None = None) -> float:
    """Critical-path completion time under a cost model (schedule.py:356-386).
    1F1B with unit costs: 2n + 2D - 2."""
    costs = costs or CostModel()
    scale = 1.0 / tl.micro_per_mini
    finish: dict[tuple, float] = {}
    ready = [0.0] * tl.depth
    end_all = 0.0
    for e in tl.events:
        start = ready[e.stage]
        dur = 0.0
        if e.kind == FORWARD:
            dur = costs.fcost(e.stage) * scale
            if e.stage > 0:
                start = max(start, finish[(FORWARD, e.mb, e.micro, e.stage - 1)])
        elif e.kind == BACKWARD:
            dur = costs.bcost(e.stage) * scale
            start = max(start, finish[(FORWARD, e.mb, e.micro, e.stage)])
            if e.stage < tl.depth - 1:
                start = max(start, finish[(BACKWARD, e.mb, e.micro, e.stage + 1)])
        end = start + dur
        finish[(e.kind, e.mb, e.micro, e.stage)] = end
        ready[e.stage] = end
        end_all = max(end_all, end)
    return end_all


# ---- export (schedule.py:391-430) ----------------------------------------------------------


def timeline_rows(tl: Timeline) -> list[dict]:
    return [dict(slot=e.slot, stage=e.stage, kind=e.kind, mb=e.mb, micro=e.micro) for e in tl.events]


def timeline_csv_text(tl: Timeline) -> str:
    body = [f"{e.slot},{e.stage},{e.kind},{e.mb},{e.micro}" for e in tl.events]
    return "\n".join([TIMELINE_CSV_HEADER, *body]) + "\n"


def timeline_json_obj(tl: Timeline) -> dict:
    return dict(
        kind=tl.kind,
        depth=tl.depth,
        n_batches=tl.n_batches,
        micro_per_mini=tl.micro_per_mini,
        horizon=tl.horizon,
        events=timeline_rows(tl),
    )


def timeline_from_json_obj(obj: dict) -> Timeline:
    evs = [ScheduleEvent(r["slot"], r["stage"], r["kind"], r["mb"], r["micro"]) for r in obj["events"]]
    return Timeline(obj["kind"], obj["depth"], obj["n_batches"], obj["micro_per_mini"], evs)


def timeline_json_text(tl: Timeline) -> str:
    return json.dumps(timeline_json_obj(tl), indent=2, sort_keys=True) + "\n"


# ---- per-stage programs for the distributed runner ------------------------------------------


@dataclass(frozen=True)
class StageOp:
    """One entry of a stage's program.

    kind/mb/micro as the timeline event; `gap` is the prediction step count s
    for this forward (None for other kinds); `fuse_predict` on an UPDATE means
    the very next op on this stage is the forward of `next_mb` with gap
    `next_gap`, so the update can be fused with that forward's prediction (K3).
    """

    kind: str
    mb: int
    micro: int = 0
    gap: int | None = None
    fuse_predict: bool = False
    next_mb: int | None = None
    next_gap: int | None = None


def stage_program(tl: Timeline, stage: int, predictive: bool = True) -> list[StageOp]:
    """Stage `stage`'s ops in execution order (== tl.stage_events(stage)).

    For predictive strategies on a non-last stage, forwards carry their gap s
    and every update immediately followed by a forward is marked for K3
    fusion (in 1F1B steady state, U_j is always followed by F_{j+D-k}).
    """
    gaps = update_gaps(tl) if predictive else {}
    evs = tl.stage_events(stage)
    last = stage == tl.depth - 1
    ops = []
    for i, e in enumerate(evs):
        gap = None
        if e.kind == FORWARD and predictive and not last:
            gap = gaps[(e.mb, stage)]
        fuse, nmb, ngap = False, None, None
        if e.kind == UPDATE and predictive and not last and i + 1 < len(evs):
            nxt = evs[i + 1]
            if nxt.kind == FORWARD and nxt.micro == 0:
                fuse, nmb, ngap = True, nxt.mb, gaps[(nxt.mb, stage)]
        ops.append(StageOp(e.kind, e.mb, e.micro, gap, fuse, nmb, ngap))
    return ops
