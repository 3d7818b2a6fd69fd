"""The weight-gradient GEMM with the optimizer update in its epilogue
(po_wgrad_update, csrc/pipeoptim_wgrad.cu: tcgen05 MMAs on bf16x3-split fp32
operands, accumulator from TMEM straight into K2/K3).

Parity: the gradient it computes (g_out) is within 2e-6 inf-norm-relative of
the float64 product x^T @ dpre (the bar of the fp32 stage GEMMs), and W', m',
v', W_hat are BIT-identical to the streaming K3 / K2 (po_step_predict /
po_step) applied to that same fp32 gradient — so the update rule itself
keeps the bit-exact contract of the K-kernels (vs the fp32 emulation) and
the <= 1e-6 one vs float64."""

import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SHAPES = [(128, 256, 128), (128, 3072, 1024), (32, 128, 256), (80, 384, 256), (16, 128, 128), (48, 256, 64)]


def _lib():
    from paper_2312_00839_b200 import _lib

    return _lib.load()


def _hp(kind):
    from paper_2312_00839_b200.optim import OptimizerConfig

    return OptimizerConfig(kind).hparams()


def _inputs(rows, fin, fout, seed):
    import torch

    g = torch.Generator(device="cuda").manual_seed(seed)
    x = torch.randn(rows, fin, device="cuda", generator=g)
    dp = torch.randn(rows, fout, device="cuda", generator=g) * 0.01
    w = torch.randn(fin, fout, device="cuda", generator=g) * 0.02
    m = torch.randn(fin, fout, device="cuda", generator=g) * 1e-3
    v = (torch.randn(fin, fout, device="cuda", generator=g) * 1e-2).square_()
    return x, dp, w, m, v


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "x".join(map(str, s)))
@pytest.mark.parametrize("kind", ["sgdm", "adam", "adamw"])
@pytest.mark.parametrize("predict", [True, False])
def test_fused_wgrad_update_matches_gemm_and_k3(shape, kind, predict):
    import torch

    lib = _lib()
    rows, fin, fout = shape
    assert lib.po_wgrad_update_supported(rows, fin, fout) == 1
    x, dp, w, m, v = _inputs(rows, fin, fout, seed=rows + fin)
    H = ctypes.byref(_hp(kind))
    s = torch.cuda.current_stream().cuda_stream
    step, lr, c_pred = 4, 1e-3, 3e-3 if predict else 0.0
    w1, m1, v1 = w.clone(), m.clone(), v.clone()
    what1 = torch.empty_like(w)
    g = torch.empty_like(w)
    bad = torch.full((1,), 2 ** 63 - 1, dtype=torch.int64, device="cuda")
    s2 = None if kind == "sgdm" else v1.data_ptr()
    rc = lib.po_wgrad_update(H, x.data_ptr(), fin, dp.data_ptr(), fout, rows, fin, fout, w1.data_ptr(), m1.data_ptr(),
                             s2, what1.data_ptr() if predict else None, g.data_ptr(), lr, c_pred, step, None,
                             bad.data_ptr(), 0, s)
    assert rc == 0, lib.po_strerror(rc)
    torch.cuda.synchronize()
    # the GEMM: within the fp32 stage-GEMM bar of the float64 product
    ref = x.double().T @ dp.double()
    err = float((g.double() - ref).abs().max() / ref.abs().max())
    assert err <= 2e-6, err
    # the update: bit-identical to the streaming kernel on the same gradient
    w2, m2, v2 = w.clone(), m.clone(), v.clone()
    what2 = torch.empty_like(w)
    s2b = None if kind == "sgdm" else v2.data_ptr()
    if predict:
        rc = lib.po_step_predict(H, w2.data_ptr(), g.data_ptr(), m2.data_ptr(), s2b, what2.data_ptr(), w.numel(), lr,
                                 c_pred, step, None, None, s)
    else:
        rc = lib.po_step(H, w2.data_ptr(), g.data_ptr(), m2.data_ptr(), s2b, None, w.numel(), lr, step, None, None, s)
    assert rc == 0
    torch.cuda.synchronize()
    assert torch.equal(w1, w2) and torch.equal(m1, m2)
    if kind != "sgdm":
        assert torch.equal(v1, v2)
    if predict:
        assert torch.equal(what1, what2)
    assert int(bad.item()) == 2 ** 63 - 1


def test_fused_wgrad_update_without_g_out_and_device_coefficients():
    """g_out NULL (the production form) and coefficients from a device
    po_coef (CUDA-graph replays) give the same update."""
    import torch

    from paper_2312_00839_b200 import _lib as L

    lib = _lib()
    rows, fin, fout = 128, 512, 256
    x, dp, w, m, v = _inputs(rows, fin, fout, seed=9)
    hp = _hp("adam")
    s = torch.cuda.current_stream().cuda_stream
    outs = []
    for dev_coef in (False, True):
        w1, m1, v1, wh = w.clone(), m.clone(), v.clone(), torch.empty_like(w)
        coef = None
        if dev_coef:
            c = torch.zeros(4, dtype=torch.float32, device="cuda")
            host = L.po_coef()
            assert lib.po_coef_fill(ctypes.byref(hp), L.PO_COEF_STEP_PREDICT, 1e-3, 2e-3, 6, ctypes.byref(host)) == 0
            c.copy_(torch.tensor([host.lr, host.c_pred, host.inv_bc1, host.inv_bc2]))
            coef = c.data_ptr()
        rc = lib.po_wgrad_update(ctypes.byref(hp), x.data_ptr(), fin, dp.data_ptr(), fout, rows, fin, fout,
                                 w1.data_ptr(), m1.data_ptr(), v1.data_ptr(), wh.data_ptr(), None,
                                 0.0 if dev_coef else 1e-3, 0.0 if dev_coef else 2e-3, 0 if dev_coef else 6, coef,
                                 None, 0, s)
        assert rc == 0
        outs.append((w1, m1, v1, wh))
    torch.cuda.synchronize()
    for a, b in zip(*outs):
        assert torch.equal(a, b)


def test_fused_wgrad_update_flags_nonfinite_and_rejects_shapes():
    import torch

    lib = _lib()
    rows, fin, fout = 32, 256, 128
    x, dp, w, m, v = _inputs(rows, fin, fout, seed=3)
    x[5, 130] = float("inf")  # poisons row 130 of the gradient
    bad = torch.full((1,), 2 ** 63 - 1, dtype=torch.int64, device="cuda")
    H = ctypes.byref(_hp("adam"))
    s = torch.cuda.current_stream().cuda_stream
    rc = lib.po_wgrad_update(H, x.data_ptr(), fin, dp.data_ptr(), fout, rows, fin, fout, w.data_ptr(), m.data_ptr(),
                             v.data_ptr(), None, None, 1e-3, 0.0, 1, None, bad.data_ptr(), 1000, s)
    assert rc == 0
    torch.cuda.synchronize()
    assert int(bad.item()) == 1000 + 130 * fout  # first non-finite element, flat offset added
    for r, i, o in ((8, 128, 128), (128, 100, 128), (128, 128, 96), (0, 128, 128)):
        assert lib.po_wgrad_update_supported(r, i, o) == 0
        assert lib.po_wgrad_update(H, x.data_ptr(), i, dp.data_ptr(), o, r, i, o, w.data_ptr(), m.data_ptr(),
                                   v.data_ptr(), None, None, 1e-3, 0.0, 1, None, None, 0, s) != 0


def _mlp_run(fuse, graphed, strategy="optimizer_prediction", kind="adam", n=12):
    import torch

    from paper_2312_00839_b200 import stages as S
    from paper_2312_00839_b200.bench_pipeline import DeviceBatches
    from paper_2312_00839_b200.optim import OptimizerConfig, OptimizerState
    from paper_2312_00839_b200.runtime import GraphedExecute, build_timeline, execute
    from paper_2312_00839_b200.stages import build_layers, build_stages, torch_init

    dev = torch.device("cuda", 0)
    dims, acts = [512, 256, 384, 128, 10], ["relu", "relu", "relu", "linear"]
    data = DeviceBatches(torch, dev, dims=dims)
    old = S.FUSE_WGRAD_UPDATE
    S.FUSE_WGRAD_UPDATE = fuse
    try:
        stages = build_stages(build_layers(dims, acts), 4, torch_init(11, dev), device=dev)
        opts = [OptimizerState(OptimizerConfig(kind), s.param_names, device=dev) for s in stages]
        tl = build_timeline(strategy, 4, n)
        if graphed:
            g = GraphedExecute(tl, stages, opts, strategy, data, "softmax_xent", lambda mb: 1e-3, streams="stage")
            reps = []
            for _ in range(2):
                g.replay()
                reps.append(g.report())
            rep = reps[-1]
        else:
            rep = execute(tl, stages, opts, strategy, data, "softmax_xent", lambda mb: 1e-3, streams="stage",
                          checks="eager")
        torch.cuda.synchronize()
        return rep, [s.flat.data.double().cpu() for s in stages]
    finally:
        S.FUSE_WGRAD_UPDATE = old


@pytest.mark.parametrize("graphed", [False, True])
@pytest.mark.parametrize("strategy,kind", [("optimizer_prediction", "adam"), ("async_raw", "adamw"),
                                           ("optimizer_prediction", "sgdm")])
def test_runner_with_fused_wgrad_matches_unfused(graphed, strategy, kind):
    """The runner with the weight gradients formed inside the update
    (stages.FUSE_WGRAD_UPDATE, step_fused_: po_wgrad_update + K2/K3 on the
    bias segments, eager and CUDA-graph replays with CoefTape scalars) ==
    the GEMM + K2/K3 path: version records exact, losses and weights equal
    up to the GEMMs' fp32 summation order. (Adam normalises each gradient
    element by its own history, so elements whose gradients are ~1e-9 of the
    largest can move by ~lr on a last-bit difference: the weight bar is 5e-4
    of the tensor's max for Adam/AdamW, 1e-6 for SGDM.)"""
    from test_runtime_gpu import rec_tuples

    a, wa = _mlp_run(False, graphed, strategy, kind)
    b, wb = _mlp_run(True, graphed, strategy, kind)
    assert rec_tuples(a) == rec_tuples(b)
    assert np.allclose(a.losses, b.losses, rtol=1e-4, atol=1e-7)
    tol = 1e-6 if kind == "sgdm" else 5e-4
    for x, y in zip(wa, wb):
        assert float((x - y).abs().max() / y.abs().max()) <= tol
