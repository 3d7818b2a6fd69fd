"""The peer-memory 1F1B runner (peer_pipeline.PeerStageRunner) with the REAL
kernels: several processes on one B200 map each other's rings over CUDA IPC
(NVLink peer memory on a multi-GPU node). Eager runs must reproduce the
reference (records exact, losses/params vs the oracle); a run captured into
ONE CUDA graph per rank and replayed must continue training exactly like
further single-process runs of the same stages."""

import json
import os
import socket
from pathlib import Path

import numpy as np
import pytest

from oracle import optim_ref, rng_ref, runtime_ref

pytestmark = pytest.mark.gpu

DIMS = [16, 24, 24, 24, 20, 10]
ACTS = ["tanh", "tanh", "relu", "tanh", "linear"]
ROWS = 8


class DevSrc:
    """Reference-seeded batches, resident on the device (graph replays read them)."""

    def __init__(self, dev):
        import torch

        self.b = {}
        for mb in range(1, 64):
            s = rng_ref.Stream(7, f"batch-{mb}")
            x, y = s.normal(ROWS, DIMS[0]), s.normal(ROWS, DIMS[-1])
            self.b[mb] = (torch.tensor(np.asarray(getattr(x, "a", x)), dtype=torch.float32, device=dev),
                          torch.tensor(np.asarray(getattr(y, "a", y)), dtype=torch.float32, device=dev))

    def batch(self, mb):
        return self.b[mb]


def _stage(rank, world, kind, dev):
    from paper_2312_00839_b200.optim import OptimizerConfig, OptimizerState
    from paper_2312_00839_b200.stages import StageModel, build_layers, partition_layers

    group = partition_layers(build_layers(DIMS, ACTS), world)[rank]
    stage = StageModel(rank, group, lambda sp: rng_ref.layer_init(3, sp.index, sp.in_dim, sp.out_dim), dev)
    kw = {"weight_decay": 0.0} if kind == "sgdm" else {}
    return stage, OptimizerState(OptimizerConfig(kind, **kw), stage.param_names, device=dev)


def _worker(rank, world, port, strategy, kind, n, replays, out_dir):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2312_00839_b200.peer_pipeline import PeerStageRunner
        from paper_2312_00839_b200.pipeline import gather_reports
        from paper_2312_00839_b200.runtime import build_timeline

        torch.backends.cuda.matmul.allow_tf32 = False
        dev = torch.device("cuda", 0)
        stage, opt = _stage(rank, world, kind, dev)
        tl = build_timeline(strategy, world, n)
        runner = PeerStageRunner(dist, tl, stage, opt, strategy, DevSrc(dev), "mse", lambda mb: 0.01, ROWS,
                                 timeout_ms=120_000)
        reps = [runner.run()]
        if replays:
            runner.capture()
            for _ in range(replays):
                runner.replay()
                reps.append(runner.report())
        allr = gather_reports(dist, reps[0], world)
        lastr = gather_reports(dist, reps[-1], world)
        if rank == 0:
            Path(out_dir, "out.json").write_text(json.dumps({
                "records": sorted([[r.mb, r.micro, r.stage, r.forward_version, r.predicted, r.prediction_target,
                                    r.backward_version, r.live_backward_version] for rp in allr for r in rp.records]),
                "losses_first": allr[-1].losses, "losses_last": lastr[-1].losses,
                "executed": [[list(e) for e in rp.executed] for rp in allr]}))
        Path(out_dir, f"params{rank}.json").write_text(json.dumps(
            {n_: p.detach().double().cpu().numpy().tolist() for n_, p in zip(stage.param_names, stage.params)}))
    finally:
        dist.destroy_process_group()


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("strategy,kind", [("optimizer_prediction", "adam"), ("async_raw", "sgdm"),
                                           ("spectrain", "sgdm")])
def test_peer_runner_eager_matches_reference(tmp_path, world, strategy, kind):
    import torch.multiprocessing as mp

    from paper_2312_00839_b200.runtime import build_timeline

    n = 2 * world + 3
    mp.spawn(_worker, args=(world, _port(), strategy, kind, n, 0, str(tmp_path)), nprocs=world, join=True)
    got = json.loads((tmp_path / "out.json").read_text())
    src = DevSrc("cpu")
    ref = runtime_ref.run(DIMS, ACTS, world, n, strategy, optim_ref.Hyper(kind, weight_decay=0.0),
                          lambda mb: tuple(t.numpy() for t in src.batch(mb)), "mse", lambda mb: 0.01,
                          lambda i, a, b: rng_ref.layer_init(3, i, a, b))
    tl = build_timeline(strategy, world, n)
    assert [[tuple(e) for e in ex] for ex in got["executed"]] == [
        [(e.kind, e.mb) for e in tl.stage_events(k)] for k in range(world)]
    assert got["records"] == sorted(list(r) for r in ref["records"])
    assert np.allclose(got["losses_first"], ref["losses"], rtol=1e-4, atol=1e-6)
    for k in range(world):
        params = json.loads((tmp_path / f"params{k}.json").read_text())
        for name, want in zip(ref["names"][k], ref["params"][k]):
            assert optim_ref.inf_norm_rel(np.array(params[name]), want) <= 1e-4


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("strategy,kind", [("optimizer_prediction", "adam"), ("async_raw", "adamw")])
def test_peer_runner_graph_replays_continue_training(tmp_path, world, strategy, kind):
    """eager run + capture + 2 replays (one CUDA graph per rank, no host in the
    loop) == 3 runs of the single-process runner on the same stages."""
    import torch
    import torch.multiprocessing as mp

    from paper_2312_00839_b200.runtime import build_timeline, execute

    n = 2 * world + 2
    mp.spawn(_worker, args=(world, _port(), strategy, kind, n, 2, str(tmp_path)), nprocs=world, join=True)
    got = json.loads((tmp_path / "out.json").read_text())
    torch.backends.cuda.matmul.allow_tf32 = False
    dev = torch.device("cuda", 0)
    pairs = [_stage(k, world, kind, dev) for k in range(world)]
    stages, opts = [p[0] for p in pairs], [p[1] for p in pairs]
    tl = build_timeline(strategy, world, n)
    src = DevSrc(dev)
    for _ in range(3):
        for s in stages:
            s.version = 1
        rep = execute(tl, stages, opts, strategy, src, "mse", lambda mb: 0.01, checks="deferred")
    np.testing.assert_allclose(got["losses_last"], rep.losses, rtol=1e-6, atol=1e-9)
    for k, st in enumerate(stages):
        params = json.loads((tmp_path / f"params{k}.json").read_text())
        for name, p in zip(st.param_names, st.params):
            want = p.detach().double().cpu().numpy()
            assert optim_ref.inf_norm_rel(np.array(params[name]), want) <= 1e-6


def _module_worker(rank, world, port, n, out_dir):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2312_00839_b200.bench_pipeline import MODULE_CONFIGS, ModuleBatches, module_stages_for
        from paper_2312_00839_b200.optim import OptimizerConfig, OptimizerState
        from paper_2312_00839_b200.peer_pipeline import PeerStageRunner
        from paper_2312_00839_b200.pipeline import gather_reports
        from paper_2312_00839_b200.runtime import build_timeline

        torch.backends.cudnn.deterministic = True
        torch.backends.cudnn.allow_tf32 = torch.backends.cuda.matmul.allow_tf32 = False
        dev = torch.device("cuda", 0)
        cfg = dict(MODULE_CONFIGS["config2_vgg16"], batch=8)
        torch.manual_seed(0)
        stages, _ = module_stages_for(torch, "config2_vgg16", dev, depth=world, costs=[1.0] * 15)
        stage = stages[rank]
        opt = OptimizerState(OptimizerConfig("sgdm"), stage.param_names, device=dev)
        tl = build_timeline("optimizer_prediction", world, n)
        runner = PeerStageRunner(dist, tl, stage, opt, "optimizer_prediction", ModuleBatches(torch, dev, cfg),
                                 "softmax_xent", lambda mb: 1e-2, 8, timeout_ms=120_000)
        runner.run()
        runner.capture()
        runner.replay()
        reps = gather_reports(dist, runner.report(), world)
        if rank == 0:
            Path(out_dir, "out.json").write_text(json.dumps({"losses": reps[-1].losses}))
        torch.save(stage.flat.data.cpu(), Path(out_dir, f"w{rank}.pt"))
    finally:
        dist.destroy_process_group()


def test_peer_runner_module_stages(tmp_path):
    """VGG-16 module stages (conv/BN/LiveLinear) through the peer runner, one
    graph per rank: eager run + 1 replay == 2 single-process runs."""
    import torch
    import torch.multiprocessing as mp

    from paper_2312_00839_b200.bench_pipeline import MODULE_CONFIGS, ModuleBatches, module_stages_for
    from paper_2312_00839_b200.optim import OptimizerConfig, OptimizerState
    from paper_2312_00839_b200.runtime import build_timeline, execute

    world, n = 2, 5
    mp.spawn(_module_worker, args=(world, _port(), n, str(tmp_path)), nprocs=world, join=True)
    got = json.loads((tmp_path / "out.json").read_text())
    torch.backends.cudnn.deterministic = True
    torch.backends.cudnn.allow_tf32 = torch.backends.cuda.matmul.allow_tf32 = False
    dev = torch.device("cuda", 0)
    cfg = dict(MODULE_CONFIGS["config2_vgg16"], batch=8)
    torch.manual_seed(0)
    stages, _ = module_stages_for(torch, "config2_vgg16", dev, depth=world, costs=[1.0] * 15)
    opts = [OptimizerState(OptimizerConfig("sgdm"), s.param_names, device=dev) for s in stages]
    tl = build_timeline("optimizer_prediction", world, n)
    data = ModuleBatches(torch, dev, cfg)
    for _ in range(2):
        for s in stages:
            s.version = 1
        rep = execute(tl, stages, opts, "optimizer_prediction", data, "softmax_xent", lambda mb: 1e-2,
                      checks="deferred")
    np.testing.assert_allclose(got["losses"], rep.losses, rtol=1e-5, atol=1e-7)
    for k, st in enumerate(stages):
        w = torch.load(tmp_path / f"w{k}.pt")
        assert float((w - st.flat.data.cpu()).abs().max()) <= 1e-5 * float(st.flat.data.abs().max())


HDIMS = [16, 24, 24, 24, 10]
HACTS = ["tanh", "tanh", "tanh", "linear"]


class HSrc:
    """Device-resident reference-seeded batches of 8 rows (DP shards them)."""

    def __init__(self, dev):
        import torch

        self.b = {}
        for mb in range(1, 64):
            s = rng_ref.Stream(9, f"batch-{mb}")
            x, y = s.normal(8, HDIMS[0]), s.normal(8, HDIMS[-1])
            self.b[mb] = (torch.tensor(np.asarray(getattr(x, "a", x)), dtype=torch.float32, device=dev),
                          torch.tensor(np.asarray(getattr(y, "a", y)), dtype=torch.float32, device=dev))

    def batch(self, mb):
        return self.b[mb]


def _hybrid_worker(rank, world, port, dp, pp, n, kind, out_dir, dp_mode="peer_load"):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2312_00839_b200.dp_fused import FusedDPGroup
        from paper_2312_00839_b200.optim import OptimizerConfig, OptimizerState
        from paper_2312_00839_b200.peer_pipeline import PeerStageRunner
        from paper_2312_00839_b200.pipeline import gather_reports
        from paper_2312_00839_b200.runtime import build_timeline
        from paper_2312_00839_b200.stages import StageModel, build_layers, partition_layers

        torch.backends.cuda.matmul.allow_tf32 = False
        dev = torch.device("cuda", 0)
        r, k = divmod(rank, pp)
        groups = [dist.new_group([q * pp + s for q in range(dp)]) for s in range(pp)]
        kw = {"weight_decay": 0.0} if kind == "sgdm" else {}
        data = HSrc(dev)
        out = {}
        for mode in ("graph", "eager"):
            stage = StageModel(k, partition_layers(build_layers(HDIMS, HACTS), pp)[k],
                               lambda sp: rng_ref.layer_init(4, sp.index, sp.in_dim, sp.out_dim), dev)
            opt = OptimizerState(OptimizerConfig(kind, **kw), stage.param_names, device=dev)
            fused = FusedDPGroup(dist, groups[k], r, dp, stage.flat.layout.numel, dev, timeout_ms=120_000,
                                 mode=dp_mode)
            runner = PeerStageRunner(dist, build_timeline("optimizer_prediction", pp, n), stage, opt,
                                     "optimizer_prediction", data, "mse", lambda mb: 0.01, 8 // dp,
                                     stage_ranks=[r * pp + s for s in range(pp)], dp_rank=r, dp_size=dp,
                                     fused_dp=fused, timeout_ms=120_000)
            reps = [runner.run()]
            if mode == "graph":
                runner.capture()
                for _ in range(2):
                    runner.replay()
                    reps.append(runner.report())
            else:
                for _ in range(2):
                    reps.append(runner.run())
            first = gather_reports(dist, reps[0], world)
            out[mode] = {"first_losses": np.mean([rp.losses for rp in first if rp.rank == pp - 1], axis=0).tolist(),
                         "params": {n_: p.detach().double().cpu().numpy().tolist()
                                    for n_, p in zip(stage.param_names, stage.params)}}
        Path(out_dir, f"h{rank}.json").write_text(json.dumps(out))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("dp_mode", ["peer_load", "shard"])
@pytest.mark.parametrize("kind", ["adam", "sgdm"])
def test_peer_runner_hybrid_dp_graph(tmp_path, kind, dp_mode):
    """DP 2 x PP 2 (4 processes on one GPU) through the peer runner with the
    DP mean fused into K3 on device epochs: the first run equals the
    full-batch 2-stage oracle pipeline, replicas stay bit-identical, and an
    eager run + capture + 2 replays equals 3 eager runs bit for bit."""
    import torch.multiprocessing as mp

    dp, pp, n = 2, 2, 8
    mp.spawn(_hybrid_worker, args=(dp * pp, _port(), dp, pp, n, kind, str(tmp_path), dp_mode), nprocs=dp * pp,
             join=True)
    res = [json.loads((tmp_path / f"h{i}.json").read_text()) for i in range(dp * pp)]
    ref = runtime_ref.run(HDIMS, HACTS, pp, n, "optimizer_prediction", optim_ref.Hyper(kind, weight_decay=0.0),
                          lambda mb: tuple(t.cpu().numpy() for t in HSrc("cpu").batch(mb)), "mse", lambda mb: 0.01,
                          lambda i, a, b: rng_ref.layer_init(4, i, a, b))
    assert np.allclose(res[0]["eager"]["first_losses"], ref["losses"], rtol=1e-4, atol=1e-6)
    for k in range(pp):
        a, b = res[k], res[pp + k]  # replicas 0 and 1 of stage k
        assert a["graph"]["params"] == b["graph"]["params"]
        assert a["graph"]["params"] == a["eager"]["params"]
