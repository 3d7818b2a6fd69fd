"""The distributed 1F1B runner with the REAL device kernels: several processes
on one B200 (the gpurun box has one GPU), gloo transport with host staging.
Covers everything of the NCCL path except NCCL itself: per-rank programs,
grouped exchanges, K1/K2/K3 on each rank's stage, deferred checks, version
records vs the oracle, losses vs the oracle."""

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


class Src:
    def batch(self, mb):
        s = rng_ref.Stream(7, f"batch-{mb}")
        return s.normal(8, DIMS[0]), s.normal(8, DIMS[-1])


def _worker(rank, world, port, strategy, kind, n, out_dir, graphed=False):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2312_00839_b200.optim import OptimizerConfig, OptimizerState
        from paper_2312_00839_b200.pipeline import PipelineStageRunner, gather_reports
        from paper_2312_00839_b200.runtime import build_timeline
        from paper_2312_00839_b200.stages import StageModel, build_layers, partition_layers

        torch.backends.cuda.matmul.allow_tf32 = False
        dev = torch.device("cuda", 0)
        group = partition_layers(build_layers(DIMS, ACTS), world)[rank]
        stage = StageModel(rank, group, lambda sp: rng_ref.layer_init(3, sp.index, sp.in_dim, sp.out_dim), dev)
        kw = {"weight_decay": 0.0} if kind == "sgdm" else {}
        opt = OptimizerState(OptimizerConfig(kind, **kw), stage.param_names, device=dev)
        tl = build_timeline(strategy, world, n)
        runner = PipelineStageRunner(dist, tl, stage, opt, strategy, Src(), "mse", lambda mb: 0.01, 8,
                                     host_staging=True, checks="deferred", graphed=graphed)
        assert (runner._graphs is not None) == graphed
        rep = runner.run()
        reps = gather_reports(dist, rep, world)
        if rank == 0:
            Path(out_dir, "out.json").write_text(json.dumps({
                "records": sorted([[r.mb, r.micro, r.stage, r.forward_version, r.predicted, r.prediction_target,
                                    r.backward_version, r.live_backward_version] for rp in reps for r in rp.records]),
                "losses": reps[-1].losses,
                "executed": [[list(e) for e in rp.executed] for rp in reps]}))
        Path(out_dir, f"params{rank}.json").write_text(json.dumps(
            {n_: p.detach().double().cpu().numpy().tolist() for n_, p in zip(stage.param_names, stage.params)}))
    finally:
        dist.destroy_process_group()


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("strategy,kind", [("optimizer_prediction", "adam"), ("async_raw", "sgdm")])
@pytest.mark.parametrize("graphed", [False, True])
def test_multiprocess_runner_with_device_kernels(tmp_path, world, strategy, kind, graphed):
    """graphed=True: every op's device work replayed from per-(kind, slot)
    CUDA graphs, optimizer scalars from the slot tape — same numbers."""
    import torch.multiprocessing as mp

    n = 3 * world + 5  # enough mini-batches that every slot is captured and replayed
    mp.spawn(_worker, args=(world, _port(), strategy, kind, n, str(tmp_path), graphed), nprocs=world, join=True)
    got = json.loads((tmp_path / "out.json").read_text())
    ref = runtime_ref.run(DIMS, ACTS, world, n, strategy, optim_ref.Hyper(kind, weight_decay=0.0), Src().batch,
                          "mse", lambda mb: 0.01, lambda i, a, b: rng_ref.layer_init(3, i, a, b))
    assert got["records"] == sorted(list(r) for r in ref["records"])
    assert np.allclose(got["losses"], ref["losses"], rtol=1e-4, atol=1e-6)
    for k in range(world):
        params = json.loads((tmp_path / f"params{k}.json").read_text())
        for name, want in zip(ref["names"][k], ref["params"][k]):
            assert optim_ref.inf_norm_rel(np.array(params[name]), want) <= 1e-4
