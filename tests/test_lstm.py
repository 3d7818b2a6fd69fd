"""LiveLSTM (GNMT stages): cuBLAS GEMMs + the po_lstm_cell_* kernels, with the
reference's stage semantics — forward on the weights given (W_hat), backward
through the LIVE weights (stages.py:187-209).

The reference has no LSTM, so the semantics are pinned by a float64 torch
restatement written here (`s9_lstm_ref`: test infrastructure only), itself
checked against torch autograd when forward and live weights coincide; the
CUDA path is checked against it, and against cuDNN's nn.LSTM (same weights,
TF32 off) as the plain fp32 reference of the same op.
"""

import pytest
import torch


def s9_lstm_ref(x, fwd, live, dy):
    """float64 LSTM layer: forward with `fwd` = (w_ih, w_hh, b_ih, b_hh),
    backward of <y, dy> with the stashed activations and the `live` weights
    for dx / dh. Returns y, dx, dW_ih, dW_hh, db."""
    w_ih, w_hh, b_ih, b_hh = fwd
    lw_ih, lw_hh = live[0], live[1]
    bsz, steps, _ = x.shape
    hid = w_hh.shape[1]
    h = x.new_zeros(bsz, hid)
    c = x.new_zeros(bsz, hid)
    ys, saved = [], []
    for t in range(steps):
        a = x[:, t] @ w_ih.T + b_ih + b_hh + h @ w_hh.T
        i, f, g, o = a.split(hid, dim=1)
        i, f, g, o = torch.sigmoid(i), torch.sigmoid(f), torch.tanh(g), torch.sigmoid(o)
        c_prev, h_prev = c, h
        c = f * c_prev + i * g
        h = o * torch.tanh(c)
        saved.append((i, f, g, o, c_prev, c, h_prev))
        ys.append(h)
    y = torch.stack(ys, 1)
    dx = torch.zeros_like(x)
    gw_ih, gw_hh = torch.zeros_like(w_ih), torch.zeros_like(w_hh)
    gb = torch.zeros_like(b_ih)
    dh_next = x.new_zeros(bsz, hid)
    dc = x.new_zeros(bsz, hid)
    for t in range(steps - 1, -1, -1):
        i, f, g, o, c_prev, c, h_prev = saved[t]
        dh = dy[:, t] + dh_next
        tc = torch.tanh(c)
        dct = dc + dh * o * (1 - tc * tc)
        da = torch.cat([dct * g * i * (1 - i), dct * c_prev * f * (1 - f), dct * i * (1 - g * g),
                        dh * tc * o * (1 - o)], 1)
        dc = dct * f
        dh_next = da @ lw_hh
        dx[:, t] = da @ lw_ih
        gw_ih += da.T @ x[:, t]
        gw_hh += da.T @ h_prev
        gb += da.sum(0)
    return y, dx, gw_ih, gw_hh, gb


def _weights(d_in, hid, seed, scale=None):
    g = torch.Generator().manual_seed(seed)
    s = scale if scale is not None else hid ** -0.5
    return [(torch.rand(shape, generator=g, dtype=torch.float64) * 2 - 1) * s
            for shape in ((4 * hid, d_in), (4 * hid, hid), (4 * hid,), (4 * hid,))]


def test_reference_matches_autograd_when_weights_coincide():
    """The float64 restatement == torch autograd through the same recurrence
    (forward weights == live weights)."""
    torch.manual_seed(0)
    bsz, steps, d_in, hid = 3, 5, 6, 4
    x = torch.randn(bsz, steps, d_in, dtype=torch.float64, requires_grad=True)
    ws = [w.requires_grad_(True) for w in _weights(d_in, hid, 1)]
    dy = torch.randn(bsz, steps, hid, dtype=torch.float64)
    h = torch.zeros(bsz, hid, dtype=torch.float64)
    c = torch.zeros(bsz, hid, dtype=torch.float64)
    ys = []
    for t in range(steps):
        a = x[:, t] @ ws[0].T + ws[2] + ws[3] + h @ ws[1].T
        i, f, g, o = a.split(hid, 1)
        c = torch.sigmoid(f) * c + torch.sigmoid(i) * torch.tanh(g)
        h = torch.sigmoid(o) * torch.tanh(c)
        ys.append(h)
    y = torch.stack(ys, 1)
    y.backward(dy)
    ry, rdx, rgi, rgh, rgb = s9_lstm_ref(x.detach(), [w.detach() for w in ws], [w.detach() for w in ws], dy)
    torch.testing.assert_close(ry, y.detach(), rtol=1e-12, atol=1e-12)
    torch.testing.assert_close(rdx, x.grad, rtol=1e-12, atol=1e-12)
    torch.testing.assert_close(rgi, ws[0].grad, rtol=1e-12, atol=1e-12)
    torch.testing.assert_close(rgh, ws[1].grad, rtol=1e-12, atol=1e-12)
    torch.testing.assert_close(rgb, ws[2].grad, rtol=1e-12, atol=1e-12)
    torch.testing.assert_close(rgb, ws[3].grad, rtol=1e-12, atol=1e-12)


def test_live_lstm_params_mirror_nn_lstm():
    from paper_2312_00839_b200.stage_models import LiveLSTM

    m, ref = LiveLSTM(12, 8), torch.nn.LSTM(12, 8, batch_first=True)
    assert [n for n, _ in m.named_parameters()] == [n for n, _ in ref.named_parameters()]
    assert [p.shape for p in m.parameters()] == [p.shape for p in ref.parameters()]
    assert all(float(p.abs().max()) <= 8 ** -0.5 for p in m.parameters())


def test_live_lstm_has_no_cpu_path():
    from paper_2312_00839_b200.stage_models import LiveLSTM

    with pytest.raises(RuntimeError, match="no CPU path"):
        LiveLSTM(4, 4)(torch.zeros(2, 3, 4))


def _rel(a, b):
    return float((a.double() - b).abs().max() / b.abs().max().clamp_min(1e-30))


@pytest.mark.gpu
@pytest.mark.parametrize("bsz,steps,d_in,hid", [(1, 1, 4, 4), (3, 7, 12, 16), (8, 20, 256, 256), (64, 50, 1024, 1024)])
def test_live_lstm_matches_cudnn_when_weights_coincide(bsz, steps, d_in, hid):
    """Same weights forward and backward: LiveLSTM == cuDNN nn.LSTM (fp32,
    TF32 off) within fp32 accumulation-order tolerance (2e-5 relative to the
    tensor's max; both are fp32 evaluations of the same recurrence)."""
    from paper_2312_00839_b200.stage_models import LiveLSTM

    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.allow_tf32 = False
    dev = torch.device("cuda", 0)
    torch.manual_seed(3)
    m = LiveLSTM(d_in, hid).to(dev)
    ref = torch.nn.LSTM(d_in, hid, batch_first=True).to(dev)
    with torch.no_grad():
        for p, q in zip(ref.parameters(), m.parameters()):
            p.copy_(q)
    x = torch.randn(bsz, steps, d_in, device=dev)
    dy = torch.randn(bsz, steps, hid, device=dev)
    xa, xb = x.clone().requires_grad_(True), x.clone().requires_grad_(True)
    ya, _ = m(xa)
    yb, _ = ref(xb)
    ya.backward(dy)
    yb.backward(dy)
    assert _rel(ya, yb.double()) < 2e-5
    assert _rel(xa.grad, xb.grad.double()) < 2e-5
    for p, q in zip(m.parameters(), ref.parameters()):
        assert _rel(p.grad, q.grad.double()) < 2e-5, p.shape


@pytest.mark.gpu
@pytest.mark.parametrize("bsz,steps,d_in,hid", [(4, 9, 8, 12), (16, 30, 128, 64), (8, 5, 256, 1024)])
def test_live_lstm_backward_uses_live_weights(bsz, steps, d_in, hid):
    """Forward on W_hat, then the parameters point back at the live buffer:
    dx / dh use the live weights, dW the stashed activations (S9). Compared
    with the float64 restatement; fp32 bar 1e-5 of the tensor's max."""
    from paper_2312_00839_b200.stage_models import LiveLSTM

    torch.backends.cuda.matmul.allow_tf32 = False
    dev = torch.device("cuda", 0)
    torch.manual_seed(5)
    m = LiveLSTM(d_in, hid).to(dev)
    fwd = [w.float() for w in _weights(d_in, hid, 7)]
    live = [w.float() for w in _weights(d_in, hid, 8)]
    params = list(m.parameters())
    fwd_d = [w.to(dev) for w in fwd]
    live_d = [w.to(dev) for w in live]
    for p, w in zip(params, fwd_d):
        p.data = w
    x = torch.randn(bsz, steps, d_in, device=dev, requires_grad=True)
    y, _ = m(x)
    for p, w in zip(params, live_d):  # the runner re-points at the live buffer
        p.data = w
    dy = torch.randn(bsz, steps, hid, device=dev)
    y.backward(dy)
    ry, rdx, rgi, rgh, rgb = s9_lstm_ref(x.detach().double().cpu(), [w.double() for w in fwd],
                                         [w.double() for w in live], dy.double().cpu())
    assert _rel(y.detach().cpu(), ry) < 1e-5
    assert _rel(x.grad.cpu(), rdx) < 1e-5
    assert _rel(params[0].grad.cpu(), rgi) < 1e-5
    assert _rel(params[1].grad.cpu(), rgh) < 1e-5
    assert _rel(params[2].grad.cpu(), rgb) < 1e-5 and _rel(params[3].grad.cpu(), rgb) < 1e-5
    # and the live weights really mattered: the forward-weight backward differs
    _, fdx, _, _, _ = s9_lstm_ref(x.detach().double().cpu(), [w.double() for w in fwd],
                                  [w.double() for w in fwd], dy.double().cpu())
    assert _rel(x.grad.cpu(), fdx) > 1e-2


@pytest.mark.gpu
def test_lstm_cell_abi_rejects_bad_shapes():
    from paper_2312_00839_b200 import _lib

    lib = _lib.load()
    t = torch.zeros(64, device="cuda")
    p = t.data_ptr()
    assert lib.po_lstm_cell_fwd(p, None, p, p, None, 0, 1, 6, None) == _lib.PO_EINVAL  # hidden % 4
    assert lib.po_lstm_cell_fwd(p + 4, None, p, p, None, 0, 1, 4, None) == _lib.PO_EINVAL  # misaligned
    assert lib.po_lstm_cell_bwd(p, None, p, p, 2, None, p, p, 1, 4, None) == _lib.PO_EINVAL  # dy_ld < hidden
    assert lib.po_lstm_cell_bwd(p, None, p, None, 0, None, p, p, 0, 4, None) == _lib.PO_EINVAL  # batch
