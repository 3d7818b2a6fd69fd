"""The narrow output layer kernels (po_head_fwd / po_head_bwd,
csrc/pipeoptim_head.cu) that replace the library GEMMs for linear layers with
<= 32 outputs (config 1's classifier): forward, input / weight / bias
gradients vs float64 (the fp32 stage-GEMM bar, 2e-6 of the max), the
accumulate form (GPipe micro-batches), the finiteness flag, determinism."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _lib():
    from paper_2312_00839_b200 import _lib

    return _lib.load()


@pytest.mark.parametrize("rows,fin,c", [(128, 1024, 10), (8, 6, 3), (300, 257, 32), (64, 1024, 1), (33, 64, 17),
                                        (512, 512, 10)])
def test_head_forward_backward_vs_float64(rows, fin, c):
    import torch

    lib = _lib()
    g0 = torch.Generator(device="cuda").manual_seed(rows + fin + c)
    x = torch.randn(rows, fin, device="cuda", generator=g0)
    w = torch.randn(fin, c, device="cuda", generator=g0) * 0.05
    b = torch.randn(c, device="cuda", generator=g0)
    g = torch.randn(rows, c, device="cuda", generator=g0) * 0.01
    s = torch.cuda.current_stream().cuda_stream
    out = torch.empty(rows, c, device="cuda")
    flags = torch.ones(1, dtype=torch.uint8, device="cuda")
    assert lib.po_head_fwd(x.data_ptr(), rows, fin, w.data_ptr(), b.data_ptr(), c, out.data_ptr(), flags.data_ptr(),
                           0, s) == 0
    dx = torch.empty(rows, fin, device="cuda")
    dw = torch.empty(fin, c, device="cuda")
    db = torch.empty(c, device="cuda")
    assert lib.po_head_bwd(x.data_ptr(), rows, fin, g.data_ptr(), c, w.data_ptr(), dx.data_ptr(), dw.data_ptr(),
                           db.data_ptr(), 0, s) == 0
    torch.cuda.synchronize()
    X, W, B, G = (t.double() for t in (x, w, b, g))

    def rel(a, ref):
        return float((a.double() - ref).abs().max() / ref.abs().max())

    assert rel(out, X @ W + B) <= 2e-6
    assert rel(dx, G @ W.T) <= 2e-6
    assert rel(dw, X.T @ G) <= 2e-6
    assert rel(db, G.sum(0)) <= 2e-6
    assert int(flags.item()) == 1
    # accumulate (micro-batch sums): adds onto what is there
    dw2, db2 = dw.clone(), db.clone()
    assert lib.po_head_bwd(x.data_ptr(), rows, fin, g.data_ptr(), c, w.data_ptr(), None, dw2.data_ptr(),
                           db2.data_ptr(), 1, s) == 0
    torch.cuda.synchronize()
    assert rel(dw2, 2 * X.T @ G) <= 2e-6 and rel(db2, 2 * G.sum(0)) <= 2e-6
    # deterministic: a second run gives the same bits
    dw3 = torch.empty_like(dw)
    db3 = torch.empty_like(db)
    assert lib.po_head_bwd(x.data_ptr(), rows, fin, g.data_ptr(), c, w.data_ptr(), None, dw3.data_ptr(),
                           db3.data_ptr(), 0, s) == 0
    torch.cuda.synchronize()
    assert torch.equal(dw3, dw) and torch.equal(db3, db)


def test_head_flags_nonfinite_and_rejects_wide_layers():
    import torch

    lib = _lib()
    x = torch.randn(4, 64, device="cuda")
    x[2, 5] = float("nan")
    w = torch.randn(64, 10, device="cuda")
    out = torch.empty(4, 10, device="cuda")
    flags = torch.ones(3, dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    assert lib.po_head_fwd(x.data_ptr(), 4, 64, w.data_ptr(), None, 10, out.data_ptr(), flags.data_ptr(), 1, s) == 0
    torch.cuda.synchronize()
    assert flags.tolist() == [1, 0, 1]
    assert lib.po_head_supported(4, 64, 33) == 0
    assert lib.po_head_fwd(x.data_ptr(), 4, 64, w.data_ptr(), None, 33, out.data_ptr(), None, 0, s) != 0


def test_stage_with_head_matches_library_path():
    """An MLP stage whose last layer is narrow: stages.FUSED_HEAD on vs off
    give the same forward output, input gradient and parameter gradients up
    to summation order."""
    import torch

    from paper_2312_00839_b200 import stages as S
    from paper_2312_00839_b200.stages import StageModel, build_layers, partition_layers, torch_init

    dev = torch.device("cuda", 0)
    x = torch.randn(128, 1024, device=dev)
    gout = torch.randn(128, 10, device=dev) * 0.01
    res = {}
    for fused in (False, True):
        S.FUSED_HEAD = fused
        try:
            st = StageModel(0, partition_layers(build_layers([1024, 10], ["linear"]), 1)[0], torch_init(2, dev), dev)
            out = st.run_forward(st.params, (1, 0), x, 1, check_finite=True)
            gin, _ = st.run_backward(st.params, (1, 0), gout, need_input_grad=True)
            torch.cuda.synchronize()
            res[fused] = (out.double(), gin.double(), st.flat.grad.double().clone())
        finally:
            S.FUSED_HEAD = True
    for a, b in zip(res[False], res[True]):
        assert float((a - b).abs().max() / b.abs().max()) <= 2e-6


@pytest.mark.parametrize("kind", ["softmax_xent", "mse"])
@pytest.mark.parametrize("rows,fin,c", [(128, 1024, 10), (1, 6, 3), (300, 257, 32), (64, 1024, 1), (33, 64, 17),
                                        (513, 512, 10)])
def test_head_fwd_loss_is_bit_identical_to_two_launches(kind, rows, fin, c):
    """po_head_fwd_loss (forward + loss + dL/dout in one launch) gives the
    same bits as po_head_fwd followed by po_loss_grad: output, gradient,
    scalar loss, finiteness flag; the scratch counter re-arms (two launches
    in a row, and a CUDA-graph replay)."""
    import torch

    from paper_2312_00839_b200 import _lib as L

    lib = _lib()
    code = L.PO_LOSS_MSE if kind == "mse" else L.PO_LOSS_SOFTMAX_XENT
    g0 = torch.Generator(device="cuda").manual_seed(rows * 7 + fin + c)
    x = torch.randn(rows, fin, device="cuda", generator=g0)
    w = torch.randn(fin, c, device="cuda", generator=g0) * 0.05
    b = torch.randn(c, device="cuda", generator=g0)
    if kind == "mse":
        y = torch.randn(rows, c, device="cuda", generator=g0)
    else:
        y = torch.nn.functional.one_hot(torch.randint(0, c, (rows,), device="cuda", generator=g0), c).float()
    s = torch.cuda.current_stream().cuda_stream

    def two():
        out, grad = torch.empty(rows, c, device="cuda"), torch.empty(rows, c, device="cuda")
        loss, scratch = torch.empty((), device="cuda"), torch.zeros(rows + 1, device="cuda")
        flags = torch.ones(1, dtype=torch.uint8, device="cuda")
        assert lib.po_head_fwd(x.data_ptr(), rows, fin, w.data_ptr(), b.data_ptr(), c, out.data_ptr(),
                               flags.data_ptr(), 0, s) == 0
        assert lib.po_loss_grad(code, out.data_ptr(), y.data_ptr(), rows, c, grad.data_ptr(), loss.data_ptr(),
                                scratch.data_ptr(), s) == 0
        return out, grad, loss, flags

    scratch = torch.zeros(rows + 1, device="cuda")
    out, grad = torch.empty(rows, c, device="cuda"), torch.empty(rows, c, device="cuda")
    loss = torch.empty((), device="cuda")
    flags = torch.ones(1, dtype=torch.uint8, device="cuda")

    def one():
        assert lib.po_head_fwd_loss(x.data_ptr(), rows, fin, w.data_ptr(), b.data_ptr(), c, y.data_ptr(), code,
                                    out.data_ptr(), grad.data_ptr(), loss.data_ptr(), scratch.data_ptr(),
                                    flags.data_ptr(), 0, torch.cuda.current_stream().cuda_stream) == 0

    want = two()
    for _ in range(2):  # the counter re-arms
        loss.fill_(float("nan"))
        one()
        torch.cuda.synchronize()
        for got, ref in zip((out, grad, loss, flags), want):
            assert torch.equal(got, ref), (kind, rows, fin, c)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        one()
    loss.fill_(float("nan"))
    graph.replay()
    torch.cuda.synchronize()
    assert torch.equal(loss, want[2]) and torch.equal(grad, want[1])


def test_head_fwd_loss_rejects_bad_arguments():
    import torch

    lib = _lib()
    p = torch.zeros(64, device="cuda").data_ptr()
    s = torch.cuda.current_stream().cuda_stream
    assert lib.po_head_fwd_loss(p, 4, 4, p, None, 2, p, 7, p, p, p, p, None, 0, s) != 0  # loss kind
    assert lib.po_head_fwd_loss(p, 4, 4, p, None, 2, None, 0, p, p, p, p, None, 0, s) != 0  # no target
    assert lib.po_head_fwd_loss(p, 4, 4, p, None, 2, p, 0, p, p, p, None, None, 0, s) != 0  # no scratch
    assert lib.po_head_fwd_loss(p, 4, 4, p, None, 33, p, 0, p, p, p, p, None, 0, s) != 0  # too wide


@pytest.mark.parametrize("kind", ["softmax_xent", "mse"])
def test_run_forward_loss_fused_equals_unfused(kind):
    """StageModel.run_forward_loss with stages.FUSED_HEAD_LOSS on (one launch)
    and off (run_forward + loss_and_grad): identical output, loss, gradient;
    a target the fused kernel cannot take (float64) falls back."""
    import torch

    from paper_2312_00839_b200 import stages as S
    from paper_2312_00839_b200.stages import StageModel, build_layers, partition_layers, torch_init

    dev = torch.device("cuda", 0)
    x = torch.randn(128, 1024, device=dev)
    y = torch.nn.functional.one_hot(torch.arange(128, device=dev) % 10, 10).float()
    if kind == "mse":
        y = y * 0.5 + 0.1
    res = {}
    for fused in (False, True):
        S.FUSED_HEAD_LOSS = fused
        try:
            st = StageModel(1, partition_layers(build_layers([512, 1024, 10], ["relu", "linear"]), 2)[1],
                            torch_init(3, dev), dev)
            res[fused] = st.run_forward_loss(st.params, (1, 0), x, 1, y, kind, check_finite=True)
            res[(fused, "f64")] = st.run_forward_loss(st.params, (2, 0), x, 1, y.double(), kind, check_finite=True)
        finally:
            S.FUSED_HEAD_LOSS = True
    torch.cuda.synchronize()
    for a, b in zip(res[False], res[True]):
        assert torch.equal(a, b)
    for a, b in zip(res[(False, "f64")], res[(True, "f64")]):
        assert torch.equal(a, b)
