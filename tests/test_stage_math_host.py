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


def test_staging_in_gradient_only_where_exact():
    """runtime.staging_in_grad_ok: W_hat may live in the gradient's storage
    only for predictive 1F1B, one micro-batch, MLP stages, switch on."""
    import numpy as np

    from paper_2312_00839_b200 import runtime
    from paper_2312_00839_b200.stages import StageModel, build_layers, partition_layers

    st = StageModel(0, partition_layers(build_layers([4, 3, 2], ["relu", "linear"]), 1)[0],
                    lambda sp: (np.zeros((sp.in_dim, sp.out_dim)), np.zeros((1, sp.out_dim))), "cpu")
    assert runtime.staging_in_grad_ok(st, True, 1)
    assert not runtime.staging_in_grad_ok(st, False, 1)  # live policies never predict
    assert not runtime.staging_in_grad_ok(st, True, 4)  # micro-batches accumulate into the gradient
    assert not runtime.staging_in_grad_ok(object(), True, 1)  # module stages may save weight views
    runtime.STAGING_IN_GRAD = False
    try:
        assert not runtime.staging_in_grad_ok(st, True, 1)
    finally:
        runtime.STAGING_IN_GRAD = True
    rt = runtime._StageRt(st, None, 1, alias_grad=True)
    assert rt.staging_buffer() is st.flat.grad
    st.set_grad_buffer(st.flat.grad.clone())  # follows a re-pointed gradient
    assert rt.staging_buffer() is st.flat.grad
