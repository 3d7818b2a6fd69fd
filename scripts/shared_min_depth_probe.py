"""Stage-concurrent config-1 runs at D = 2 and 3 with the shared-GPU
policies (runtime.SHARED_GPU_*) on vs off (runtime.SHARED_GPU_MIN_DEPTH),
graphed, the arms alternated (median of 5)."""
import json
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2312_00839_b200 import bench_pipeline as bp  # noqa: E402
from paper_2312_00839_b200 import runtime  # noqa: E402
from paper_2312_00839_b200.optim import OptimizerConfig, OptimizerState  # noqa: E402
from paper_2312_00839_b200.runtime import GraphedExecute, build_timeline  # noqa: E402
from paper_2312_00839_b200.stages import build_layers, build_stages, torch_init  # noqa: E402

torch.backends.cuda.matmul.allow_tf32 = False
dev = torch.device("cuda", 0)
data = bp.DeviceBatches(torch, dev)
n = 64
graphs = {}
for depth in (2, 3):
    for policy in ("latency", "shared"):
        runtime.SHARED_GPU_MIN_DEPTH = depth if policy == "shared" else 4
        for strategy in ("async_raw", "optimizer_prediction"):
            st = build_stages(build_layers(bp.CONFIG1_DIMS, bp.CONFIG1_ACTS), depth, torch_init(0, dev), device=dev)
            opts = [OptimizerState(OptimizerConfig("adam"), s.param_names, device=dev) for s in st]
            g = GraphedExecute(build_timeline(strategy, depth, n), st, opts, strategy, data, "softmax_xent",
                               lambda mb: 1e-4, warmup_runs=1, streams="stage")
            g.replay()
            graphs[(depth, policy, strategy)] = (g, st, opts)
runtime.SHARED_GPU_MIN_DEPTH = 4
torch.cuda.synchronize()
times = {k: [] for k in graphs}
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _ in range(5):
    for k, (g, _, _) in graphs.items():
        e0.record()
        for _ in range(3):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        times[k].append(e0.elapsed_time(e1) / 3e3)
for depth in (2, 3):
    for policy in ("latency", "shared"):
        off = n * bp.BATCH / statistics.median(times[(depth, policy, "async_raw")])
        on = n * bp.BATCH / statistics.median(times[(depth, policy, "optimizer_prediction")])
        print(json.dumps({"depth": depth, "policy": policy, "pred_off": round(off), "pred_on": round(on),
                          "overhead": round(1 - on / off, 4)}), flush=True)
