"""Debug driver: the graphed distributed runner, N processes sharing one GPU
(gloo + host staging) with a short gloo timeout so a hang becomes a traceback."""
import datetime
import os
import socket
import sys
import traceback
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))


def worker(rank, world, port, strategy, kind, n, graphed):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world, timeout=datetime.timedelta(seconds=60))
    try:
        from oracle import rng_ref
        from paper_2312_00839_b200.optim import OptimizerConfig, OptimizerState
        from paper_2312_00839_b200.pipeline import PipelineStageRunner
        from paper_2312_00839_b200.runtime import build_timeline
        from paper_2312_00839_b200.stages import StageModel, build_layers, partition_layers
        from test_pipeline_gpu_multiproc import ACTS, DIMS, Src

        dev = torch.device("cuda", 0)
        group = partition_layers(build_layers(DIMS, ACTS), world)[rank]
        stage = StageModel(rank, group, lambda sp: rng_ref.layer_init(3, sp.index, sp.in_dim, sp.out_dim), dev)
        opt = OptimizerState(OptimizerConfig(kind), stage.param_names, device=dev)
        runner = PipelineStageRunner(dist, build_timeline(strategy, world, n), stage, opt, strategy, Src(), "mse",
                                     lambda mb: 0.01, 8, host_staging=True, checks="deferred", graphed=graphed)
        if os.environ.get("PO_TRACE"):
            orig_f, orig_b, orig_u = runner._graphs.forward, runner._graphs.backward, runner._graphs.update

            def tf(op, *a):
                print(f"[r{rank}] F{op.mb} count={dict(runner._graphs.count)}", flush=True)
                return orig_f(op, *a)

            def tb(op, *a):
                print(f"[r{rank}] B{op.mb}", flush=True)
                return orig_b(op, *a)

            def tu(op):
                print(f"[r{rank}] U{op.mb}", flush=True)
                return orig_u(op)

            runner._graphs.forward, runner._graphs.backward, runner._graphs.update = tf, tb, tu
        rep = runner.run()
        print(f"[r{rank}] done losses={rep.losses[:3] if rep.losses else None}", flush=True)
    except Exception:
        print(f"[r{rank}] EXC", traceback.format_exc(), flush=True)
        os._exit(1)
    finally:
        dist.destroy_process_group()


if __name__ == "__main__":
    import torch.multiprocessing as mp

    world = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    strategy = sys.argv[2] if len(sys.argv) > 2 else "optimizer_prediction"
    kind = sys.argv[3] if len(sys.argv) > 3 else "adam"
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mp.spawn(worker, args=(world, port, strategy, kind, 3 * world + 5, True), nprocs=world, join=True)
