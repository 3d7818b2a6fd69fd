"""The one-process-per-GPU 1F1B runner's host logic (per-rank programs,
grouped neighbour exchanges, version bookkeeping, loss/record collection) on
CPU with the gloo backend and world_size 2 and 4.

The device kernels are not available on CPU, so these tests give the runner a
torch stand-in optimizer defined HERE (the reference formulas in fp64 torch
ops) — test infrastructure only; the product path has no CPU optimizer.
The B200 run of the same runner over NCCL is covered by bench.py --gpus N.
"""

import json
import os
import socket
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import optim_ref, rng_ref, runtime_ref

DIMS = [4, 6, 6, 6, 6, 5, 3]
ACTS = ["tanh"] * 5 + ["linear"]


class StandInOptimizer:
    """CPU stand-in exposing the runner-facing surface of OptimizerState
    (step_ / predict_ / step_predict_ / check_finite) in float64 torch."""

    def __init__(self, kind, names, lr_eps=1e-8):
        self.kind, self.names = kind, names
        self.config = optim_ref.Hyper(kind, weight_decay=0.0)
        self.step_count = 0
        self.eager_checks = False
        self.s1 = self.s2 = None

    def _dir(self, t):
        h = self.config
        if self.kind == "sgdm":
            return self.s1
        bc1, bc2 = 1.0 - h.beta1 ** t, 1.0 - h.beta2 ** t
        return (self.s1 / bc1) / (torch.sqrt(self.s2 / bc2) + h.eps)

    def step_(self, flat, lr):
        h = self.config
        w = flat.data.double()
        g = flat.grad.double()
        if self.s1 is None:
            self.s1 = torch.zeros_like(w)
            self.s2 = torch.zeros_like(w)
        if self.kind == "sgdm":
            self.s1 = h.momentum * self.s1 + (1.0 - h.dampening) * (g + h.weight_decay * w)
            d = self.s1
        else:
            self.s1 = h.beta1 * self.s1 + (1.0 - h.beta1) * g
            self.s2 = h.beta2 * self.s2 + (1.0 - h.beta2) * (g * g)
            d = self._dir(self.step_count + 1)
            if self.kind == "adamw":
                d = d + h.decoupled_decay * w
        flat.data.copy_(w - lr * d)
        self.step_count += 1

    def predict_(self, flat, lr, s, out):
        if self.step_count == 0:
            out.copy_(flat.data)
        else:
            out.copy_(flat.data.double() - (lr * s) * self._dir(self.step_count))

    def step_predict_(self, flat, lr, lr_pred, s, out):
        self.step_(flat, lr)
        self.predict_(flat, lr_pred, s, out)

    def check_finite(self):
        pass


class Src:
    def batch(self, mb):
        s = rng_ref.Stream(101, f"batch-{mb}")
        return s.normal(8, DIMS[0]), s.normal(8, DIMS[-1])


def _worker(rank, world, port, strategy, kind, n, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2312_00839_b200.pipeline import PipelineStageRunner, gather_reports
        from paper_2312_00839_b200.runtime import build_timeline
        from paper_2312_00839_b200.stages import StageModel, build_layers, partition_layers

        torch.set_default_dtype(torch.float32)
        layers = build_layers(DIMS, ACTS)
        group = partition_layers(layers, world)[rank]
        stage = StageModel(rank, group, lambda sp: rng_ref.layer_init(5, sp.index, sp.in_dim, sp.out_dim), "cpu")
        opt = StandInOptimizer(kind, stage.param_names)
        tl = build_timeline(strategy, world, n)
        runner = PipelineStageRunner(dist, tl, stage, opt, strategy, Src(), "mse", lambda mb: 0.01, 8)
        rep = runner.run()
        reps = gather_reports(dist, rep, world)
        if rank == 0:
            payload = {
                "records": sorted(
                    [[r.mb, r.micro, r.stage, r.forward_version, r.predicted, r.prediction_target,
                      r.backward_version, r.live_backward_version] for rp in reps for r in rp.records]),
                "executed": [[list(e) for e in rp.executed] for rp in reps],
                "losses": reps[-1].losses,
                "stash": [rp.stash_peak for rp in reps],
                "snap": [rp.snapshot_peak for rp in reps],
                "versions": [rp.final_version for rp in reps],
            }
            Path(out_dir, "out.json").write_text(json.dumps(payload))
        params = {n_: p.detach().double().numpy().tolist() for n_, p in zip(stage.param_names, stage.params)}
        Path(out_dir, f"params{rank}.json").write_text(json.dumps(params))
    finally:
        dist.destroy_process_group()


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("strategy,kind", [("optimizer_prediction", "adam"), ("optimizer_prediction", "sgdm"),
                                           ("async_raw", "adamw")])
def test_gloo_pipeline_matches_oracle(tmp_path, world, strategy, kind):
    n = 2 * world + 6
    mp.spawn(_worker, args=(world, free_port(), strategy, kind, n, str(tmp_path)), nprocs=world, join=True)
    got = json.loads((tmp_path / "out.json").read_text())
    ref = runtime_ref.run(DIMS, ACTS, world, n, strategy, optim_ref.Hyper(kind, weight_decay=0.0), Src().batch, "mse",
                          lambda mb: 0.01, lambda i, a, b: rng_ref.layer_init(5, i, a, b))
    # bit-exact bookkeeping
    assert got["records"] == sorted(list(r) for r in ref["records"])
    from paper_2312_00839_b200.runtime import build_timeline

    tl = build_timeline(strategy, world, n)
    for k in range(world):
        assert [tuple(e) for e in got["executed"][k]] == [(e.kind, e.mb) for e in tl.stage_events(k)]
    assert got["versions"] == [n + 1] * world
    assert got["stash"] == ref["stash_peaks"] and got["snap"] == ref["snapshot_peaks"]
    # numbers: fp32 stage math vs the fp64 oracle
    assert np.allclose(got["losses"], ref["losses"], rtol=1e-4, atol=1e-6)
    for k in range(world):
        params = json.loads((tmp_path / f"params{k}.json").read_text())
        for name, want in zip(ref["names"][k], ref["params"][k]):
            assert optim_ref.inf_norm_rel(np.array(params[name]), want) <= 1e-4


def _hybrid_worker(rank, world, port, dp, pp, n, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2312_00839_b200.pipeline import PipelineStageRunner, gather_reports
        from paper_2312_00839_b200.runtime import build_timeline
        from paper_2312_00839_b200.stages import StageModel, build_layers, partition_layers

        r, k = divmod(rank, pp)
        groups = [dist.new_group([q * pp + s for q in range(dp)]) for s in range(pp)]
        layers = build_layers(DIMS, ACTS)
        stage = StageModel(k, partition_layers(layers, pp)[k],
                           lambda sp: rng_ref.layer_init(5, sp.index, sp.in_dim, sp.out_dim), "cpu")
        opt = StandInOptimizer("adam", stage.param_names)
        tl = build_timeline("optimizer_prediction", pp, n)
        runner = PipelineStageRunner(dist, tl, stage, opt, "optimizer_prediction", Src(), "mse", lambda mb: 0.01,
                                     8 // dp, stage_ranks=[r * pp + s for s in range(pp)], dp_group=groups[k],
                                     dp_rank=r, dp_size=dp)
        rep = runner.run()
        reps = gather_reports(dist, rep, world)
        if rank == 0:
            last = [rp for rp in reps if rp.rank == pp - 1]
            losses = np.mean([rp.losses for rp in last], axis=0).tolist()
            Path(out_dir, "out.json").write_text(json.dumps({"losses": losses}))
        params = {n_: p.detach().double().numpy().tolist() for n_, p in zip(stage.param_names, stage.params)}
        Path(out_dir, f"params{rank}.json").write_text(json.dumps(params))
    finally:
        dist.destroy_process_group()


def test_hybrid_dp_pp_equals_full_batch_pipeline(tmp_path):
    """DP=2 x PP=2 on 4 gloo ranks (each replica half of every batch, stage
    gradients averaged before the fused update) == the 2-stage pipeline on the
    full batch (oracle), and the two replicas stay identical."""
    dp, pp, n = 2, 2, 10
    mp.spawn(_hybrid_worker, args=(dp * pp, free_port(), dp, pp, n, str(tmp_path)), nprocs=dp * pp, join=True)
    got = json.loads((tmp_path / "out.json").read_text())
    ref = runtime_ref.run(DIMS, ACTS, pp, n, "optimizer_prediction", optim_ref.Hyper("adam", weight_decay=0.0),
                          Src().batch, "mse", lambda mb: 0.01, lambda i, a, b: rng_ref.layer_init(5, i, a, b))
    assert np.allclose(got["losses"], ref["losses"], rtol=1e-4, atol=1e-6)
    for k in range(pp):
        p0 = json.loads((tmp_path / f"params{k}.json").read_text())
        p1 = json.loads((tmp_path / f"params{pp + k}.json").read_text())
        for name, want in zip(ref["names"][k], ref["params"][k]):
            assert p0[name] == p1[name]  # replicas identical
            assert optim_ref.inf_norm_rel(np.array(p0[name]), want) <= 1e-4


def _conv_worker(rank, world, port, n, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import torch.nn as nn

        from paper_2312_00839_b200.pipeline import PipelineStageRunner, gather_reports
        from paper_2312_00839_b200.runtime import build_timeline
        from paper_2312_00839_b200.stage_models import LiveLinear, build_module_stages

        torch.manual_seed(0)
        blocks = [nn.Sequential(nn.Conv2d(3, 8, 3, padding=1), nn.ReLU()),
                  nn.Sequential(nn.Conv2d(8, 8, 3, padding=1), nn.ReLU(), nn.MaxPool2d(2)),
                  nn.Sequential(nn.Flatten(), LiveLinear(8 * 4 * 4, 5))]
        stages = build_module_stages(blocks, world, "cpu", (3, 8, 8))
        stage = stages[rank]
        opt = StandInOptimizer("sgdm", stage.param_names)

        class ImgSrc:
            def batch(self, mb):
                g = torch.Generator().manual_seed(mb)
                return torch.randn(4, 3, 8, 8, generator=g), torch.nn.functional.one_hot(
                    torch.randint(0, 5, (4,), generator=g), 5).float()

        tl = build_timeline("optimizer_prediction", world, n)
        runner = PipelineStageRunner(dist, tl, stage, opt, "optimizer_prediction", ImgSrc(), "softmax_xent",
                                     lambda mb: 0.05, 4)
        rep = runner.run()
        reps = gather_reports(dist, rep, world)
        if rank == 0:
            Path(out_dir, "out.json").write_text(json.dumps({
                "records": sorted([[r.mb, r.stage, r.forward_version, r.predicted, r.prediction_target,
                                    r.backward_version, r.live_backward_version] for rp in reps for r in rp.records]),
                "losses": reps[-1].losses}))
    finally:
        dist.destroy_process_group()


def test_gloo_module_stages_pipeline(tmp_path):
    """Conv module stages (4-D activations over P2P) through the distributed runner."""
    world, n = 3, 8
    mp.spawn(_conv_worker, args=(world, free_port(), n, str(tmp_path)), nprocs=world, join=True)
    got = json.loads((tmp_path / "out.json").read_text())
    ref = runtime_ref.run([3] * (world + 1), ["tanh"] * world, world, n, "optimizer_prediction",
                          optim_ref.Hyper("sgdm"), lambda mb: (np.ones((2, 3)), np.ones((2, 3))), "mse",
                          lambda mb: 1e-3, lambda i, a, b: rng_ref.layer_init(0, i, a, b))
    want = sorted([[r[0], r[2], r[3], r[4], r[5], r[6], r[7]] for r in ref["records"]])
    assert got["records"] == want
    assert len(got["losses"]) == n and all(np.isfinite(got["losses"]))


GOLDEN_GPIPE = [c for c in json.loads((Path(__file__).resolve().parent / "golden" / "runtime_golden.json").read_text())
                if c["strategy"] == "gpipe"]


class GoldenSrc:
    """The golden runs' batches (pkg/tests/test_runtime.py:22-31 seeding)."""

    def __init__(self, case):
        self.c = case

    def batch(self, mb):
        s = rng_ref.Stream(self.c["data_seed"], f"batch-{mb}")
        return s.normal(self.c["rows"], self.c["dims"][0]), s.normal(self.c["rows"], self.c["dims"][-1])


def _gpipe_worker(rank, world, port, case, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2312_00839_b200.pipeline import PipelineStageRunner, gather_reports
        from paper_2312_00839_b200.runtime import build_timeline
        from paper_2312_00839_b200.stages import StageModel, build_layers, partition_layers

        layers = build_layers(case["dims"], case["acts"])
        stage = StageModel(rank, partition_layers(layers, world)[rank],
                           lambda sp: rng_ref.layer_init(case["init_seed"], sp.index, sp.in_dim, sp.out_dim), "cpu")
        opt = StandInOptimizer(case["kind"], stage.param_names)
        tl = build_timeline("gpipe", world, case["n"], case["micros"])
        runner = PipelineStageRunner(dist, tl, stage, opt, "gpipe", GoldenSrc(case), "mse",
                                     lambda mb, lr=case["lr"]: lr, case["rows"])
        rep = runner.run()
        reps = gather_reports(dist, rep, world)
        if rank == 0:
            Path(out_dir, "out.json").write_text(json.dumps({
                "records": sorted([[r.mb, r.micro, r.stage, r.forward_version, r.predicted, r.prediction_target,
                                    r.backward_version, r.live_backward_version] for rp in reps for r in rp.records]),
                "executed": [[list(e) for e in rp.executed] for rp in reps],
                "losses": reps[-1].losses, "versions": [rp.final_version for rp in reps]}))
        params = [p.detach().double().numpy().tolist() for p in stage.params]
        Path(out_dir, f"params{rank}.json").write_text(json.dumps(params))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case", GOLDEN_GPIPE, ids=lambda c: f"D{c['depth']}-T{c['micros']}-{c['kind']}")
def test_gloo_gpipe_matches_reference_golden(tmp_path, case):
    """§8(f)#2 on the distributed runner: GPipe (T micro-batches, gradients
    averaged over them before the update, runtime.py:441-454) over gloo at
    world = D against fixtures made by the reference's own execute."""
    world = case["depth"]
    mp.spawn(_gpipe_worker, args=(world, free_port(), case, str(tmp_path)), nprocs=world, join=True)
    got = json.loads((tmp_path / "out.json").read_text())
    assert got["records"] == sorted(case["records"])
    from paper_2312_00839_b200.runtime import build_timeline

    tl = build_timeline("gpipe", world, case["n"], case["micros"])
    for k in range(world):
        want = [(e.kind, e.mb) if case["micros"] == 1 else (e.kind, e.mb, e.micro) for e in tl.stage_events(k)]
        assert [tuple(e) for e in got["executed"][k]] == want
    assert got["versions"] == case["final_versions"]
    assert np.allclose(got["losses"], case["losses"], rtol=1e-4, atol=1e-6)
    for k in range(world):
        params = json.loads((tmp_path / f"params{k}.json").read_text())
        for p, want in zip(params, case["params"][k]):
            assert optim_ref.inf_norm_rel(np.array(p), np.array(want)) <= 1e-4


def _fd_worker(rank, world, port, out_dir):
    import os

    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2312_00839_b200.dp_fused import send_fd

        if rank == 0:
            r, w = os.pipe()
            os.write(w, b"nvls-handle")
            os.close(w)
            send_fd(dist, None, rank, world, r)
            os.close(r)
        else:
            fd = send_fd(dist, None, rank, world, None)
            data = os.read(fd, 64) if rank == 1 else b"(pipe drained by rank 1)"
            os.close(fd)
            Path(out_dir, f"fd{rank}.txt").write_bytes(data)
    finally:
        dist.destroy_process_group()


def _fd_error_worker(rank, world, port, out_dir):
    import os

    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2312_00839_b200.dp_fused import send_fd

        try:
            send_fd(dist, None, rank, world, None, error="no multicast" if rank == 0 else None)
            msg = "returned"
        except RuntimeError as exc:
            msg = str(exc)
        Path(out_dir, f"err{rank}.txt").write_text(msg)
    finally:
        dist.destroy_process_group()


def test_fd_passing_propagates_replica0_failure(tmp_path):
    """If replica 0 cannot create the handle, every replica raises its error
    instead of waiting on the socket."""
    import torch.multiprocessing as mp

    mp.spawn(_fd_error_worker, args=(3, free_port(), str(tmp_path)), nprocs=3, join=True)
    for r in range(3):
        assert "no multicast" in (tmp_path / f"err{r}.txt").read_text()


def test_fd_passing_for_nvls_handles(tmp_path):
    """dp_fused.send_fd: replica 0's POSIX fd (the NVLS multicast object's
    exported handle on a GPU box; a pipe here) reaches every other replica
    over an abstract UNIX socket (SCM_RIGHTS) — all receive the same open file."""
    import torch.multiprocessing as mp

    mp.spawn(_fd_worker, args=(3, free_port(), str(tmp_path)), nprocs=3, join=True)
    assert (tmp_path / "fd1.txt").read_bytes() == b"nvls-handle"
    assert (tmp_path / "fd2.txt").exists()
