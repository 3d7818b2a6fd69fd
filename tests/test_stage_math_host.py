"""Host-side choices of the device stage math (no GPU needed): split-K slice
counts, and the CUDA-graph capture guard."""

import gc

import pytest

from paper_2312_00839_b200.stages import _splitk, _splitk_tc


@pytest.mark.parametrize("rows,k,n,want", [(128, 3072, 1024, 8), (128, 1024, 1024, 4), (128, 1024, 10, 32),
                                           (128, 10, 1024, 1), (1024, 3072, 1024, 1), (64, 1024, 4096, 4),
                                           (64, 4096, 1024, 8)])
def test_simt_split_counts(rows, k, n, want):
    s = _splitk(rows, k, n)
    assert s == want and k % s == 0


@pytest.mark.parametrize("rows,k,want", [(128, 3072, 8), (128, 1024, 8), (128, 384, 2), (128, 128, 1),
                                         (1024, 3072, 1), (8, 256, 2)])
def test_tensor_core_split_counts(rows, k, want):
    s = _splitk_tc(rows, k)
    assert s == want and k % s == 0 and (s == 1 or k // s >= 128)


def test_capture_guard_collects_and_disables_gc(monkeypatch):
    """runtime.capture: a full collection before, automatic GC off during,
    restored after (a mid-capture collection destroyed older graphs)."""
    import contextlib

    import torch

    from paper_2312_00839_b200 import runtime

    seen = {}

    @contextlib.contextmanager
    def fake_graph(graph, capture_error_mode="global"):
        seen["mode"] = capture_error_mode
        seen["enabled_inside"] = gc.isenabled()
        yield

    monkeypatch.setattr(torch.cuda, "graph", fake_graph)
    assert gc.isenabled()
    with runtime.capture(object()):
        pass
    assert seen == {"mode": "thread_local", "enabled_inside": False}
    assert gc.isenabled()
