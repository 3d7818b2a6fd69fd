"""Stage-concurrent single-GPU runner: `execute(..., streams="stage")` puts
each stage's events on its own CUDA stream (the D-GPU pipeline's concurrency
on one device). Each stage's arithmetic and its order are unchanged, so every
run must be BIT-identical to the serial runner — and through it to the
reference goldens (records exact, losses in tolerance)."""

import pytest

from test_runtime_gpu import CONFIG1, EXTRA, SMALL, build, check_losses, rec_tuples, run_case  # noqa: F401

pytestmark = pytest.mark.gpu


def _run(case, streams, checks="eager", fuse=True, gemm_split_cap=None, gemm_tile_n=None):
    from oracle import data_ref
    from paper_2312_00839_b200.runtime import execute
    from test_runtime_gpu import ArraySource, Source

    tl, stages, opts = build(case)
    if case["name"].startswith("small"):
        src, loss = Source(case["data_seed"], case["rows"], case["dims"][0], case["dims"][-1]), "mse"
    else:
        batches, loss = data_ref.config1(seed=case["data_seed"])
        src = ArraySource(batches)
    rep = execute(tl, stages, opts, case["strategy"], src, loss, lambda mb, lr=case["lr"]: lr,
                  checks=checks, fuse=fuse, streams=streams, gemm_split_cap=gemm_split_cap,
                  gemm_tile_n=gemm_tile_n)
    return rep, stages


def _same(a, sa, b, sb):
    import torch

    assert a.losses == b.losses
    assert rec_tuples(a) == rec_tuples(b)
    assert a.snapshot_peaks == b.snapshot_peaks and a.stash_peaks == b.stash_peaks
    for x, y in zip(sa, sb):
        assert torch.equal(x.flat.data, y.flat.data)


@pytest.mark.parametrize("case", SMALL + EXTRA,
                         ids=lambda c: f"D{c['depth']}-{c['strategy']}-T{c.get('micros', 1)}-{c['kind']}")
def test_stage_streams_bit_identical_to_serial(case):
    a, sa = _run(case, "serial")
    b, sb = _run(case, "stage")
    _same(a, sa, b, sb)
    assert rec_tuples(b) == case["records"]
    check_losses(b.losses, case["losses"])


@pytest.mark.parametrize("case", CONFIG1, ids=lambda c: c["strategy"])
def test_config1_stage_streams_host_batches(case):
    """Host (numpy) batches: x and y are staged to the device on stage 0's
    stream and consumed by the last stage's. Under one GEMM policy (split
    cap, tile width) the two runners agree bit for bit: the stage runner's
    default (the shared-GPU policy: 4 slices, 128-wide tiles) == the serial
    runner under it, and both runners under the latency policy (8, 64)
    agree too; either policy meets the reference goldens."""
    from paper_2312_00839_b200 import runtime

    a, sa = _run(case, "serial", checks="deferred", gemm_split_cap=runtime.SHARED_GPU_SPLIT_CAP,
                 gemm_tile_n=runtime.SHARED_GPU_GEMM_TILE_N)
    b, sb = _run(case, "stage", checks="deferred")
    _same(a, sa, b, sb)
    c, sc = _run(case, "serial", checks="deferred")
    d, sd = _run(case, "stage", checks="deferred", gemm_split_cap=8, gemm_tile_n=64)
    _same(c, sc, d, sd)
    assert rec_tuples(b) == case["records"] and rec_tuples(c) == case["records"]
    for rep in (b, c):
        check_losses(rep.losses[:10], case["losses"][:10])
        check_losses(rep.losses, case["losses"], rtol=5e-3)


def test_gemm_split_cap_context():
    """stages.gemm_split_cap bounds the tensor-core GEMM's K slices and
    restores the previous cap; non-powers of two are refused."""
    from paper_2312_00839_b200 import stages as S

    assert S._splitk_tc(128, 3072) == 8
    with S.gemm_split_cap(4):
        assert S._splitk_tc(128, 3072) == 4 and S._splitk_tc(128, 256) == 2
        with S.gemm_split_cap(1):
            assert S._splitk_tc(128, 3072) == 1
        assert S._splitk_tc(128, 3072) == 4
    assert S._splitk_tc(128, 3072) == 8
    with pytest.raises(ValueError):
        with S.gemm_split_cap(3):
            pass


def test_stage_streams_unfused_and_eager_checks():
    case = next(c for c in SMALL if c["depth"] == 4 and c["strategy"] == "optimizer_prediction"
                and c["kind"] == "adam")
    a, sa = _run(case, "serial", fuse=False)
    b, sb = _run(case, "stage", fuse=False)
    _same(a, sa, b, sb)
    c, sc = _run(case, "stage", checks="deferred")
    assert c.losses == b.losses


@pytest.mark.parametrize("strategy,kind", [("optimizer_prediction", "adam"), ("async_raw", "adamw"),
                                           ("weight_stashing", "sgdm")])
def test_graphed_stage_streams_equal_graphed_serial(strategy, kind):
    """The multi-stream capture (fork/join inside the graph) replays to the
    same bits as the single-stream capture."""
    import torch

    from paper_2312_00839_b200.bench_pipeline import DeviceBatches
    from paper_2312_00839_b200.optim import OptimizerConfig, OptimizerState
    from paper_2312_00839_b200.runtime import GraphedExecute, build_timeline
    from paper_2312_00839_b200.stages import build_layers, build_stages, torch_init

    dev = torch.device("cuda", 0)
    dims, acts = [256, 512, 384, 256, 10], ["relu", "relu", "relu", "linear"]
    data = DeviceBatches(torch, dev, dims=dims)
    tl = build_timeline(strategy, 4, 11)
    out = {}
    for streams in ("serial", "stage"):
        stages = build_stages(build_layers(dims, acts), 4, torch_init(5, dev), device=dev)
        opts = [OptimizerState(OptimizerConfig(kind), s.param_names, device=dev) for s in stages]
        g = GraphedExecute(tl, stages, opts, strategy, data, "softmax_xent", lambda mb: 1e-3, streams=streams)
        losses = []
        for _ in range(3):
            g.replay()
            losses.append(g.report().losses)
        torch.cuda.synchronize()
        out[streams] = (losses, [s.flat.data.clone() for s in stages])
    assert out["serial"][0] == out["stage"][0]
    for x, y in zip(out["serial"][1], out["stage"][1]):
        assert torch.equal(x, y)


@pytest.fixture
def separate_staging():
    """runtime.STAGING_IN_GRAD = False for the duration of a test."""
    from paper_2312_00839_b200 import runtime

    runtime.STAGING_IN_GRAD = False
    yield
    runtime.STAGING_IN_GRAD = True


def _run_both(case, streams, fuse=True, checks="eager"):
    from paper_2312_00839_b200 import runtime

    runtime.STAGING_IN_GRAD = False
    try:
        a = _run(case, streams, checks=checks, fuse=fuse)
    finally:
        runtime.STAGING_IN_GRAD = True
    return a, _run(case, streams, checks=checks, fuse=fuse)


@pytest.mark.parametrize("case", [c for c in SMALL + CONFIG1 if c["strategy"] == "optimizer_prediction"],
                         ids=lambda c: f"{c['name']}-D{c['depth']}-{c['kind']}")
@pytest.mark.parametrize("streams,fuse", [("serial", True), ("stage", True), ("stage", False)])
def test_staging_in_gradient_storage_is_exact(case, streams, fuse):
    """W_hat written over the dead gradient (runtime.STAGING_IN_GRAD, the
    default) == a separate staging buffer, bit for bit: records, losses,
    weights — fused K3 and K1 predictions, serial and stage streams."""
    (a, sa), (b, sb) = _run_both(case, streams, fuse=fuse, checks="deferred" if case in CONFIG1 else "eager")
    _same(a, sa, b, sb)


def test_staging_in_gradient_storage_graphed(separate_staging):
    """The same for CUDA-graph replays (config-1-shaped MLP, stage streams)."""
    import torch

    from paper_2312_00839_b200 import runtime
    from paper_2312_00839_b200.bench_pipeline import DeviceBatches
    from paper_2312_00839_b200.optim import OptimizerConfig, OptimizerState
    from paper_2312_00839_b200.runtime import GraphedExecute, build_timeline
    from paper_2312_00839_b200.stages import build_layers, build_stages, torch_init

    dev = torch.device("cuda", 0)
    dims, acts = [512, 384, 384, 256, 10], ["relu", "relu", "relu", "linear"]
    data = DeviceBatches(torch, dev, dims=dims)
    tl = build_timeline("optimizer_prediction", 4, 12)
    out = {}
    for alias in (False, True):
        runtime.STAGING_IN_GRAD = alias
        stages = build_stages(build_layers(dims, acts), 4, torch_init(3, dev), device=dev)
        opts = [OptimizerState(OptimizerConfig("adam"), s.param_names, device=dev) for s in stages]
        g = GraphedExecute(tl, stages, opts, "optimizer_prediction", data, "softmax_xent", lambda mb: 1e-3,
                           streams="stage")
        losses = []
        for _ in range(3):
            g.replay()
            losses.append(g.report().losses)
        torch.cuda.synchronize()
        out[alias] = (losses, [s.flat.data.clone() for s in stages])
    assert out[False][0] == out[True][0]
    for x, y in zip(out[False][1], out[True][1]):
        assert torch.equal(x, y)


@pytest.mark.parametrize("streams", ["serial", "stage"])
def test_traced_run_device_timeline(tmp_path, streams):
    """execute(trace=True): one device-timed entry per event in the
    reference's order; within a stage (one stream) events never overlap and
    follow tl.stage_events(k); the results are those of the untraced run;
    reports.write_device_timeline writes them."""
    import torch

    from paper_2312_00839_b200 import reports
    from paper_2312_00839_b200.runtime import execute
    from test_runtime_gpu import Source

    case = next(c for c in SMALL if c["depth"] == 4 and c["strategy"] == "optimizer_prediction")
    a, sa = _run(case, streams)
    tl, stages, opts = build(case)
    src = Source(case["data_seed"], case["rows"], case["dims"][0], case["dims"][-1])
    rep = execute(tl, stages, opts, case["strategy"], src, "mse", lambda mb, lr=case["lr"]: lr, checks="eager",
                  streams=streams, trace=True)
    _same(a, sa, rep, stages)
    tlog = rep.device_timeline
    assert [(r["stage"], r["kind"], r["mb"], r["micro"]) for r in tlog] == \
        [(e.stage, e.kind, e.mb, e.micro) for e in tl.events]
    for k in range(tl.depth):
        mine = [r for r in tlog if r["stage"] == k]
        assert [(r["kind"], r["mb"]) for r in mine] == [(e.kind, e.mb) for e in tl.stage_events(k)]
        for x, y in zip(mine, mine[1:]):
            assert x["start_us"] <= x["end_us"] <= y["start_us"] + 1e-3
    out = reports.write_device_timeline(rep, tmp_path / "device_timeline.csv")
    lines = out.read_text().splitlines()
    assert lines[0] == reports.DEVICE_TIMELINE_CSV_HEADER and len(lines) == 1 + len(tl.events)
    torch.cuda.synchronize()


def test_pdl_switch_leaves_results_bit_identical():
    """po_set_pdl(1) (programmatic dependent launch of the short stream
    kernels; every kernel waits for its predecessor before touching memory)
    gives the same bits as plain launches: a config-1-shaped graphed run with
    the switch on vs off; the _lib.pdl context restores the setting."""
    import torch

    from paper_2312_00839_b200 import _lib
    from paper_2312_00839_b200.bench_pipeline import DeviceBatches
    from paper_2312_00839_b200.optim import OptimizerConfig, OptimizerState
    from paper_2312_00839_b200.runtime import GraphedExecute, build_timeline, execute
    from paper_2312_00839_b200.stages import build_layers, build_stages, torch_init

    dev = torch.device("cuda", 0)
    dims, acts = [1024, 512, 512, 10], ["relu", "relu", "linear"]
    data = DeviceBatches(torch, dev, dims=dims)
    tl = build_timeline("optimizer_prediction", 3, 9)
    assert _lib.load().po_get_pdl() == 0
    out = {}
    for on in (False, True):
        with _lib.pdl(on):
            assert _lib.load().po_get_pdl() == int(on)
            stages = build_stages(build_layers(dims, acts), 3, torch_init(2, dev), device=dev)
            opts = [OptimizerState(OptimizerConfig("adamw"), s.param_names, device=dev) for s in stages]
            rep = execute(tl, stages, opts, "optimizer_prediction", data, "softmax_xent", lambda mb: 1e-3,
                          checks="deferred")
            g = GraphedExecute(tl, stages, opts, "optimizer_prediction", data, "softmax_xent", lambda mb: 1e-3)
            g.replay()
            torch.cuda.synchronize()
            out[on] = (rep.losses, g.report().losses, [s.flat.data.clone() for s in stages])
    assert _lib.load().po_get_pdl() == 0
    assert out[False][0] == out[True][0] and out[False][1] == out[True][1]
    for x, y in zip(out[False][2], out[True][2]):
        assert torch.equal(x, y)


def test_shared_gpu_optimizer_launch_is_scoped_to_the_run():
    """With >= 4 stages sharing the GPU the runner launches the stages' K2/K3
    in its shared-GPU shape (runtime.SHARED_GPU_OPT_LAUNCH) only for the run,
    never over a caller's own launch shape; results equal a run with the
    default shape, bit for bit."""
    import torch

    from paper_2312_00839_b200 import _lib, runtime
    from paper_2312_00839_b200.bench_pipeline import DeviceBatches
    from paper_2312_00839_b200.optim import OptimizerConfig, OptimizerState
    from paper_2312_00839_b200.runtime import build_timeline, execute
    from paper_2312_00839_b200.stages import build_layers, build_stages, torch_init

    dev = torch.device("cuda", 0)
    dims, acts = [512, 384, 384, 256, 10], ["relu", "relu", "relu", "linear"]
    data = DeviceBatches(torch, dev, dims=dims)
    tl = build_timeline("optimizer_prediction", 4, 10)
    own = _lib.make_launch(256, 4, 8, 1, 1)
    out = {}
    for shape in (runtime.SHARED_GPU_OPT_LAUNCH, None):
        old = runtime.SHARED_GPU_OPT_LAUNCH
        runtime.SHARED_GPU_OPT_LAUNCH = shape
        try:
            stages = build_stages(build_layers(dims, acts), 4, torch_init(4, dev), device=dev)
            opts = [OptimizerState(OptimizerConfig("adam"), s.param_names, device=dev,
                                   launch=own if i == 1 else None) for i, s in enumerate(stages)]
            rep = execute(tl, stages, opts, "optimizer_prediction", data, "softmax_xent", lambda mb: 1e-3,
                          checks="deferred", streams="stage")
            torch.cuda.synchronize()
        finally:
            runtime.SHARED_GPU_OPT_LAUNCH = old
        assert [o._launch is None for o in opts] == [True, False, True, True]
        assert opts[1]._launch is own
        out[shape] = (rep.losses, [s.flat.data.clone() for s in stages])
    a, b = out.values()
    assert a[0] == b[0]
    for x, y in zip(a[1], b[1]):
        assert torch.equal(x, y)
