"""Deadlock freedom of the NCCL runner's posting order (pipeline.exchange_plan)
under NCCL's group semantics, checked by simulation (no GPU, no NCCL).

Model (conservative): each rank posts its grouped exchanges in order on ONE
communicator, so its groups execute one at a time, each starting only after
the previous one completed and the work op between them ran (the op needs the
previous group's receive; the next group's send needs the op's output). A
send and the matching receive — the same link, matched in posting order per
direction, as NCCL matches point-to-point ops per peer pair — complete
together only while both are in their ranks' ACTIVE groups (rendezvous: no
buffering of any message, the worst case for large activations). Ops of one
group progress independently; a group completes when all its ops have. The
run deadlocks iff at some point no active pair can complete while a rank
still has groups left. Random completion orders are explored as in
tests/test_peer_slots.py; the reference's single-threaded executor it
replaces is /root/reference/pkg/src/pipesim/runtime.py:404-466.
"""

import random

import pytest

from paper_2312_00839_b200.pipeline import exchange_plan
from paper_2312_00839_b200.schedule import build_1f1b, build_gpipe, stage_program


def _plans(depth, n, micros=None):
    tl = build_1f1b(depth, n) if micros is None else build_gpipe(depth, n, micros)
    return [exchange_plan(stage_program(tl, k, predictive=micros is None), k, depth) for k in range(depth)]


def _simulate(plans, seed):
    """True iff every rank finishes every group."""
    D = len(plans)
    rng = random.Random(seed)
    # sequence number of each message on its link, in posting order per side
    seq = [[] for _ in range(D)]
    for k, groups in enumerate(plans):
        counts = {}
        for g in groups:
            row = []
            for side, link, mb in g:
                key = (side, link)
                row.append((side, link, counts.get(key, 0), mb))
                counts[key] = counts.get(key, 0) + 1
            seq[k].append(row)
    active = [0] * D
    done = [set() for _ in range(D)]  # indices done within the active group

    def peer_of(k, link):
        kind, b = link  # boundary b is between stage b and b + 1
        return b + 1 if k == b else b

    while True:
        for k in range(D):  # retire completed groups
            while active[k] < len(seq[k]) and len(done[k]) == len(seq[k][active[k]]):
                active[k] += 1
                done[k] = set()
        if all(active[k] == len(seq[k]) for k in range(D)):
            return True
        pairs = []
        for k in range(D):
            if active[k] == len(seq[k]):
                continue
            for i, (side, link, s, mb) in enumerate(seq[k][active[k]]):
                if i in done[k] or side != "send":
                    continue
                p = peer_of(k, link)
                if active[p] == len(seq[p]):
                    continue
                for j, (pside, plink, ps, pmb) in enumerate(seq[p][active[p]]):
                    if j not in done[p] and pside == "recv" and plink == link and ps == s:
                        assert pmb == mb, "a receive would match another mini-batch's message"
                        pairs.append((k, i, p, j))
        if not pairs:
            return False
        k, i, p, j = rng.choice(pairs)
        done[k].add(i)
        done[p].add(j)


@pytest.mark.parametrize("depth", [2, 3, 4, 5, 6, 7, 8])
def test_nccl_posting_order_never_deadlocks(depth):
    for n in range(1, 3 * depth + 6):
        plans = _plans(depth, n)
        for seed in range(8):
            assert _simulate(plans, seed), (depth, n, seed)


@pytest.mark.parametrize("depth", [2, 4, 8])
@pytest.mark.parametrize("micros", [1, 2, 4])
def test_gpipe_posting_order_never_deadlocks(depth, micros):
    for n in (1, 2, 5):
        plans = _plans(depth, n, micros)
        for seed in range(4):
            assert _simulate(plans, seed), (depth, micros, n, seed)


def test_every_message_is_sent_and_received_once():
    for depth in (2, 4, 8):
        for n in (1, 5, 19):
            plans = _plans(depth, n)
            sends, recvs = [], []
            for groups in plans:
                for g in groups:
                    assert len(g) <= 2
                    sends += [(link, mb) for side, link, mb in g if side == "send"]
                    recvs += [(link, mb) for side, link, mb in g if side == "recv"]
            assert sorted(sends) == sorted(recvs)
            assert len(sends) == 2 * (depth - 1) * n


def test_simulator_detects_a_crossed_order():
    """Sanity of the model: two ranks that both send first to each other in
    separate groups before receiving deadlock under rendezvous."""
    m = (1, 0)
    a = [[("send", ("act", 0), m)], [("recv", ("grad", 0), m)]]
    b = [[("send", ("grad", 0), m)], [("recv", ("act", 0), m)]]
    assert not _simulate([a, b], 0)
    # the runner's pairing ({send a, recv g} vs {send g, recv a}) completes
    a2 = [[("send", ("act", 0), m), ("recv", ("grad", 0), m)]]
    b2 = [[("send", ("grad", 0), m), ("recv", ("act", 0), m)]]
    assert _simulate([a2, b2], 0)
