"""The reference-shaped optimizer API on the device (pkg/tests/test_optim.py,
re-run against paper_2312_00839_b200.optim). Values are fp32 on the device,
so the reference's 1e-14 fp64 tolerances become fp32-scale ones."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

FROZEN_SGDM_WD_TRAJ = [0.85, 0.5725, 0.19412499999999994]
FROZEN_SGDM_WD_V = 3.7837500000000004
FROZEN_ADAM_TRAJ = [0.400000001, 0.43661035347207483, 0.45027941967382146, 0.41086943043487656, 0.3926517886119052]
FROZEN_ADAM_DELTA_AFTER_5 = 0.18217641822971373
FROZEN_ADAMW_TRAJ = [0.98900000005, 0.9853476296701932, 0.9809579905841741]
FROZEN_ADAMW_DELTA_AFTER_3 = 0.34042914563488874
F32 = 2e-7


def T(v):
    import torch

    return torch.tensor([[float(v)]], dtype=torch.float32, device="cuda")


def run_steps(cfg, w0, gs, lr):
    from paper_2312_00839_b200.optim import OptimizerState

    st = OptimizerState(cfg, ["p"])
    params = [T(w0)]
    traj = []
    for g in gs:
        params, _ = st.step(params, [T(g)], lr)
        traj.append(float(params[0][0, 0]))
    return st, params, traj


def cfgs():
    from paper_2312_00839_b200.optim import OptimizerConfig

    return OptimizerConfig


def test_sgdm_frozen():
    C = cfgs()
    st, _, traj = run_steps(C("sgdm", momentum=0.9, weight_decay=0.5), 1.0, [1.0] * 3, 0.1)
    assert np.allclose(traj, FROZEN_SGDM_WD_TRAJ, rtol=0, atol=F32 * 4)
    assert abs(float(st.momentum_buf[0][0, 0]) - FROZEN_SGDM_WD_V) <= 4 * F32 * FROZEN_SGDM_WD_V


def test_adam_frozen_and_read():
    C = cfgs()
    st, params, traj = run_steps(C("adam"), 0.5, [1.0, -2.0, 0.5, 3.0, -1.0], 0.1)
    assert np.allclose(traj, FROZEN_ADAM_TRAJ, rtol=0, atol=1e-6)
    assert abs(float(st.prediction_direction(params)[0][0, 0]) - FROZEN_ADAM_DELTA_AFTER_5) <= 1e-6


def test_adamw_frozen_and_read_excludes_decay():
    C = cfgs()
    st, params, traj = run_steps(C("adamw", decoupled_decay=0.1), 1.0, [2.0, -1.0, 0.5], 0.01)
    assert np.allclose(traj, FROZEN_ADAMW_TRAJ, rtol=0, atol=1e-6)
    assert abs(float(st.prediction_direction(params)[0][0, 0]) - FROZEN_ADAMW_DELTA_AFTER_3) <= 1e-6


def test_degenerate_sgd_and_first_adam_step():
    C = cfgs()
    _, params, _ = run_steps(C("sgdm", momentum=0.0, weight_decay=0.0), 1.0, [0.5], 0.1)
    assert abs(float(params[0][0, 0]) - 0.95) <= F32
    from paper_2312_00839_b200.optim import OptimizerState

    st = OptimizerState(C("adam"), ["p"])
    _, dirs = st.step([T(0.0)], [T(2.0)], 0.001)
    assert abs(float(dirs[0][0, 0]) - 1.0) <= 1e-6


def test_zero_read_before_first_step_and_pure_read():
    import torch

    from paper_2312_00839_b200.optim import OptimizerState

    C = cfgs()
    for kind in ("sgdm", "adam", "adamw"):
        st = OptimizerState(C(kind), ["a", "b"])
        dirs = st.prediction_direction([torch.zeros(2, 2, device="cuda"), torch.zeros(1, 2, device="cuda")])
        assert all(float(d.abs().max()) == 0.0 for d in dirs)
    st = OptimizerState(C("adam"), ["p"])
    params, _ = st.step([T(1.0)], [T(0.7)], 0.01)
    before = (st.step_count, st.exp_avg[0].clone(), st.exp_avg_sq[0].clone())
    r1 = st.prediction_direction(params)
    r2 = st.prediction_direction(params)
    assert torch.equal(r1[0], r2[0])
    assert before[0] == st.step_count and torch.equal(before[1], st.exp_avg[0])


def test_predict_weights_values_and_linearity():
    import torch

    from paper_2312_00839_b200.optim import predict_weights

    (out,) = predict_weights([T(1.0)], 0.1, 3, [T(0.5)])
    assert abs(float(out[0, 0]) - 0.85) <= F32
    g = torch.Generator(device="cuda").manual_seed(9)
    p = [torch.randn(3, 3, device="cuda", generator=g)]
    d = [torch.randn(3, 3, device="cuda", generator=g)]
    assert torch.equal(predict_weights(p, 0.1, 0, d)[0], p[0])
    p1, p2, p3 = (predict_weights(p, 0.05, s, d)[0] for s in (1, 2, 3))
    assert float(((p2 - p1) - (p3 - p2)).abs().max()) <= 1e-6
    with pytest.raises(ValueError):
        predict_weights(p, 0.1, -1, d)
    with pytest.raises(ValueError):
        predict_weights(p, 0.1, 1, d + d)


@pytest.mark.parametrize("s", [1, 2, 3])
def test_prediction_exact_at_momentum_fixed_point(s):
    from paper_2312_00839_b200.optim import OptimizerState, predict_weights

    C = cfgs()
    u, g, lr = 0.9, 0.8, 0.05
    st = OptimizerState(C("sgdm", momentum=u, weight_decay=0.0), ["p"])
    st.momentum_buf = [T(g / (1 - u))]
    st.step_count = 1
    params = [T(2.0)]
    pred = predict_weights(params, lr, s, st.prediction_direction(params))
    walk = [T(2.0)]
    for _ in range(s):
        walk, _ = st.step(walk, [T(g)], lr)
    assert abs(float(pred[0][0, 0]) - float(walk[0][0, 0])) <= 1e-6


@pytest.mark.parametrize("kind", ["sgdm", "adam", "adamw"])
def test_telescoping(kind):
    import torch

    from paper_2312_00839_b200.optim import OptimizerState

    C = cfgs()
    gen = torch.Generator(device="cuda").manual_seed(31)
    st = OptimizerState(C(kind), ["p"])
    w0 = torch.randn(8, 8, device="cuda", generator=gen)
    params = [w0.clone()]
    total = torch.zeros(8, 8, dtype=torch.float64, device="cuda")
    for _ in range(100):
        params, dirs = st.step(params, [torch.randn(8, 8, device="cuda", generator=gen)], 0.01)
        total += dirs[0].double()
    recon = w0.double() - 0.01 * total
    assert float((recon - params[0].double()).abs().max()) <= 1e-5


@pytest.mark.parametrize("kind", ["sgdm", "adam"])
def test_applied_direction_equals_read(kind):
    import torch

    from paper_2312_00839_b200.optim import OptimizerState

    C = cfgs()
    gen = torch.Generator(device="cuda").manual_seed(13)
    st = OptimizerState(C(kind, weight_decay=0.0), ["p"])
    params = [torch.randn(4, 4, device="cuda", generator=gen)]
    for _ in range(20):
        params, dirs = st.step(params, [torch.randn(4, 4, device="cuda", generator=gen)], 0.01)
        assert torch.equal(st.prediction_direction(params)[0], dirs[0])


def test_step_aborts_on_non_finite_naming_parameter():
    from paper_2312_00839_b200.errors import NumericError
    from paper_2312_00839_b200.optim import OptimizerState

    C = cfgs()
    st = OptimizerState(C("sgdm", weight_decay=0.0), ["layer0.w", "layer2.w"])
    with pytest.raises(NumericError) as exc:
        st.step([T(1.0), T(1.0)], [T(0.0), T(float("inf"))], 0.1)
    assert "layer2.w" in str(exc.value)
    assert st.step_count == 0


def test_host_buffers_round_trip():
    """CPU tensors in, CPU tensors out: the host-buffer (end-to-end) path."""
    import torch

    from oracle import optim_ref as R
    from paper_2312_00839_b200.optim import OptimizerState

    C = cfgs()
    rng = np.random.default_rng(4)
    shapes = [(64, 33), (1, 33), (33, 10)]
    ps = [rng.normal(0, 0.05, s).astype(np.float32) for s in shapes]
    gs = [rng.normal(0, 0.01, s).astype(np.float32) for s in shapes]
    st = OptimizerState(C("adamw"), ["a", "b", "c"])
    new, dirs = st.step([torch.from_numpy(p) for p in ps], [torch.from_numpy(g) for g in gs], 1e-3)
    assert all(not t.is_cuda for t in new)
    orc = R.OracleOptimizer(R.Hyper("adamw"), ["a", "b", "c"])
    want, _ = orc.step([p.astype(np.float64) for p in ps], [g.astype(np.float64) for g in gs], 1e-3)
    for a, b in zip(new, want):
        assert R.inf_norm_rel(a.double().numpy(), b) <= 1e-6


@pytest.mark.parametrize("kind", ["sgdm", "adam"])
def test_host_streamer_paths_match_oracle(kind):
    """HostStreamer: host round trip (W, G in; W', W_hat out) and the
    device-resident variant (G in) agree with the oracle across chunk edges."""
    import torch

    from oracle import optim_ref as R
    from paper_2312_00839_b200.optim import HostStreamer, OptimizerConfig, OptimizerState

    n = (1 << 12) * 5 + 7  # several chunks + a ragged tail
    rng = np.random.default_rng(11)
    w = rng.normal(0, 0.02, n).astype(np.float32)
    gs = [rng.normal(0, 1e-2, n).astype(np.float32) for _ in range(3)]
    dev = torch.device("cuda", 0)
    st = HostStreamer(dev, chunk_elems=1 << 12, slots=3)
    cfg = OptimizerConfig(kind)
    o1 = OptimizerState(cfg, ["flat"], device=dev)
    o2 = OptimizerState(cfg, ["flat"], device=dev)
    w_h = torch.from_numpy(w.copy()).pin_memory()
    wo = torch.empty(n).pin_memory()
    wh = torch.empty(n).pin_memory()
    wd = torch.from_numpy(w.copy()).to(dev)
    whd = torch.empty(n, device=dev)
    orc = R.OracleOptimizer(R.Hyper(kind), ["w"])
    pw = [w.astype(np.float64)]
    for g in gs:
        g_h = torch.from_numpy(g).pin_memory()
        st.step_predict(o1, w_h, g_h, 1e-3, 2e-3, 3, wo, wh)
        st.step_predict_resident(o2, wd, g_h, 1e-3, 2e-3, 3, whd)
        torch.cuda.synchronize()
        w_h.copy_(wo)
        pw, _ = orc.step(pw, [g.astype(np.float64)], 1e-3)
        (want_hat,) = R.predict_weights(pw, 2e-3, 3, orc.prediction_direction(pw))
        assert R.inf_norm_rel(wo.double().numpy(), pw[0]) <= 1e-6
        assert R.inf_norm_rel(wh.double().numpy(), want_hat) <= 1e-6
        assert torch.equal(wd.cpu(), wo) and torch.equal(whd.cpu(), wh)
    assert o1.step_count == o2.step_count == 3


def test_host_list_api_streams_in_chunks():
    """The reference-shaped list API on host tensors (step -> W', dirs;
    predict_weights) goes through the chunked HostStreamer: several
    parameters, chunk edges inside and across them, a ragged tail; results
    <= 1e-6 vs the oracle and bit-exact vs the fp32 emulation; a non-finite
    update names its parameter like optim.py:82-84."""
    import torch

    from oracle import optim_f32
    from oracle import optim_ref as R
    from paper_2312_00839_b200.errors import NumericError
    from paper_2312_00839_b200.optim import (FlatLayout, HostStreamer, OptimizerConfig, OptimizerState,
                                             predict_weights)

    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(5)
    shapes = [(3, 3001), (7,), (5000,), (1,)]
    names = ["a", "b", "c", "d"]
    ps = [rng.normal(0, 0.02, s).astype(np.float32) for s in shapes]
    opt = OptimizerState(OptimizerConfig("adam"), names, device=dev)
    opt._bind(FlatLayout(names, shapes))
    opt._host_streamer = HostStreamer(dev, chunk_elems=1 << 12, slots=2)
    orc = R.OracleOptimizer(R.Hyper("adam"), names)
    cur64 = [p.astype(np.float64) for p in ps]
    cur = [torch.from_numpy(p.copy()) for p in ps]
    m = [np.zeros(s, np.float32) for s in shapes]
    v = [np.zeros(s, np.float32) for s in shapes]
    for t in range(3):
        gs = [rng.normal(0, 1e-2, s).astype(np.float32) for s in shapes]
        new, dirs = opt.step(cur, [torch.from_numpy(g) for g in gs], 1e-3)
        want, wdirs = orc.step([c.numpy().astype(np.float64) for c in cur], [g.astype(np.float64) for g in gs], 1e-3)
        for i, (a, b) in enumerate(zip(new, want)):
            assert not a.is_cuda
            assert R.inf_norm_rel(a.double().numpy(), b) <= (1e-6 if a.numel() >= 64 else 1e-5)
            ew, m[i], v[i], _ = optim_f32.step("adam", cur[i].numpy(), gs[i], m[i], v[i], 1e-3, t)
            assert np.array_equal(a.numpy(), ew)
        cur = new
        cur64 = want
    d = opt.prediction_direction(cur)
    wh = predict_weights(cur, 1e-3, 3, d)
    want_hat = R.predict_weights([c.numpy().astype(np.float64) for c in cur], 1e-3, 3,
                                   orc.prediction_direction(cur64))
    for a, b in zip(wh, want_hat):
        assert not a.is_cuda and R.inf_norm_rel(a.double().numpy(), b) <= 1e-5
    bad = [torch.from_numpy(g) for g in (np.zeros(s, np.float32) for s in shapes)]
    bad[2][4321] = float("inf")
    with pytest.raises(NumericError, match="in c"):
        opt.step(cur, bad, 1e-3)


def test_host_list_api_keeps_no_reference_to_its_outputs():
    """After step / prediction_direction / predict_weights on host lists
    return, nothing inside the library holds their tensors: outputs the
    caller drops go straight back to torch's pinned-host cache, so the next
    call reuses them instead of pinning fresh memory
    (profiles/r2_list_api_probe.jsonl)."""
    import gc
    import weakref

    import torch

    from paper_2312_00839_b200.optim import OptimizerConfig, OptimizerState, predict_weights

    dev = torch.device("cuda", 0)
    opt = OptimizerState(OptimizerConfig("adam"), ["w"], device=dev)
    w = torch.randn(10_000) * 0.02
    g = torch.randn(10_000) * 1e-2
    new, dirs = opt.step([w], [g], 1e-3)
    d = opt.prediction_direction(new)
    wh = predict_weights(new, 1e-3, 3, d)
    refs = [weakref.ref(t) for t in (new[0], dirs[0], d[0], wh[0], w, g)]
    del new, dirs, d, wh, w, g
    gc.collect()
    assert all(r() is None for r in refs)
