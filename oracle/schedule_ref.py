"""Independent restatement of the 1F1B schedule and its version gaps — TEST ORACLE.

Instead of the closed-form slot formulas (pkg/src/pipesim/schedule.py:150-172,
which paper_2312_00839_b200/schedule.py implements), this derives each
stage's program from the 1F1B RULE itself (Algorithm 1 / SPEC.md):
stage k of D runs min(D-k, n) warm-up forwards, then alternates
backward(+update) / forward until the forwards run out, then drains the
remaining backwards; every backward is followed by its update. Slots come
from the data dependencies (a unit-cost list schedule), which reproduces the
reference's slot indices; the global order sorts by (slot, stage, update
after its backward) as schedule.py:28,74.
"""

from __future__ import annotations

F, B, U = "forward", "backward", "update"


def stage_sequence(depth: int, n: int, k: int) -> list[tuple[str, int]]:
    warm = min(depth - k, n)
    seq = [(F, m) for m in range(1, warm + 1)]
    nf, nb = warm, 0
    while nb < n:
        nb += 1
        seq += [(B, nb), (U, nb)]
        if nf < n:
            nf += 1
            seq.append((F, nf))
    return seq


def gaps(depth: int, n: int) -> dict[tuple[int, int], int]:
    """(mb, stage) -> updates strictly between F_mb and B_mb on that stage."""
    out = {}
    for k in range(depth):
        seen, at_f = 0, {}
        for kind, m in stage_sequence(depth, n, k):
            if kind == U:
                seen += 1
            elif kind == F:
                at_f[m] = seen
            else:
                out[(m, k)] = seen - at_f[m]
    return out


def slots(depth: int, n: int) -> dict[tuple[str, int, int], int]:
    """Earliest-start unit-time slots honouring per-stage program order and
    the pipeline dependencies (forward after the previous stage's forward,
    backward after the next stage's backward). Updates share the slot of
    their backward."""
    progs = [stage_sequence(depth, n, k) for k in range(depth)]
    pos = [0] * depth
    free = [0] * depth  # next free slot per stage
    done: dict[tuple[str, int, int], int] = {}
    remaining = sum(len(p) for p in progs)
    while remaining:
        progressed = False
        for k in range(depth):
            while pos[k] < len(progs[k]):
                kind, m = progs[k][pos[k]]
                if kind == U:
                    done[(U, m, k)] = done[(B, m, k)]
                else:
                    deps = []
                    if kind == F and k > 0:
                        deps.append((F, m, k - 1))
                    if kind == B and k < depth - 1:
                        deps.append((B, m, k + 1))
                    if any(d not in done for d in deps):
                        break
                    start = max([free[k]] + [done[d] + 1 for d in deps])
                    done[(kind, m, k)] = start
                    free[k] = start + 1
                pos[k] += 1
                remaining -= 1
                progressed = True
        if not progressed:
            raise RuntimeError("1F1B program deadlocked")
    return done


def global_order(depth: int, n: int) -> list[tuple[int, int, str, int]]:
    """[(slot, stage, kind, mb)] in the reference's execution order."""
    sl = slots(depth, n)
    evs = [(s, k, kind, m) for (kind, m, k), s in sl.items()]
    evs.sort(key=lambda e: (e[0], e[1], 1 if e[2] == U else 0))
    return evs
