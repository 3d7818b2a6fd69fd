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
