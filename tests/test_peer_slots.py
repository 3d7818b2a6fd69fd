"""Ring sizing of the peer-memory transport (peer_pipeline.ring_slots): with
`slots` = 1 + the most messages in flight per link in the reference's global
event order, ranks running their own programs asynchronously (blocking
receives, credit-blocked sends) always complete — checked by simulating
random interleavings of the D per-rank programs."""

import random

import pytest

from paper_2312_00839_b200.peer_pipeline import ring_slots
from paper_2312_00839_b200.schedule import BACKWARD, FORWARD, UPDATE, build_1f1b, stage_program


def _simulate(tl, slots, seed):
    D = tl.depth
    progs = [stage_program(tl, k) for k in range(D)]
    pc = [0] * D
    phase = [0] * D  # 0: need input, 1: need to send output
    sent = {}  # link -> messages produced
    used = {}  # link -> messages consumed

    def link_in(k, op):
        if op.kind == FORWARD and k > 0:
            return ("act", k - 1)
        if op.kind == BACKWARD and k < D - 1:
            return ("grad", k)
        return None

    def link_out(k, op):
        if op.kind == FORWARD and k < D - 1:
            return ("act", k)
        if op.kind == BACKWARD and k > 0:
            return ("grad", k - 1)
        return None

    rng = random.Random(seed)
    while any(pc[k] < len(progs[k]) for k in range(D)):
        runnable = []
        for k in range(D):
            if pc[k] >= len(progs[k]):
                continue
            op = progs[k][pc[k]]
            if op.kind == UPDATE:
                runnable.append(k)
            elif phase[k] == 0:
                li = link_in(k, op)
                if li is None or sent.get(li, 0) > used.get(li, 0):
                    runnable.append(k)
            else:
                lo = link_out(k, op)
                if lo is None or sent.get(lo, 0) - used.get(lo, 0) < slots[lo]:
                    runnable.append(k)
        if not runnable:
            return False
        k = rng.choice(runnable)
        op = progs[k][pc[k]]
        if op.kind == UPDATE:
            pc[k] += 1
        elif phase[k] == 0:
            li = link_in(k, op)
            if li is not None:
                used[li] = used.get(li, 0) + 1
            phase[k] = 1
        else:
            lo = link_out(k, op)
            if lo is not None:
                sent[lo] = sent.get(lo, 0) + 1
            phase[k] = 0
            pc[k] += 1
    return True


@pytest.mark.parametrize("depth", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("n", [1, 2, 5, 17])
def test_ring_slots_never_deadlock(depth, n):
    tl = build_1f1b(depth, n)
    slots = ring_slots(tl)
    assert all(2 <= v <= 3 for v in slots.values())
    assert len(slots) == 2 * (depth - 1)
    for seed in range(30):
        assert _simulate(tl, slots, seed)

