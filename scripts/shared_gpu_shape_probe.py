"""Optimizer launch shape at pipeline-stage sizes when the stages share one
GPU: config-1 graphed stage-concurrent runs with every stage's K2/K3 under
the default small-N shape (128 x 16 CTAs/SM) vs fewer, larger CTAs, all
arms replayed in alternation (median of 7); then the per-stage unit times
ALONE (16-unit graphs) under the default vs the best shared shape."""
import json
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2312_00839_b200 import _lib  # noqa: E402
from paper_2312_00839_b200 import bench_pipeline as bp  # noqa: E402
from paper_2312_00839_b200.optim import OptimizerConfig, OptimizerState  # noqa: E402
from paper_2312_00839_b200.runtime import GraphedExecute, build_timeline  # noqa: E402
from paper_2312_00839_b200.stages import build_layers, build_stages, torch_init  # noqa: E402

torch.backends.cuda.matmul.allow_tf32 = False
dev = torch.device("cuda", 0)
data = bp.DeviceBatches(torch, dev)
n = 64
shapes = {"default": None, "512x2": (512, 2, 8, 1, 1), "256x4": (256, 4, 8, 1, 1), "512x1": (512, 1, 8, 1, 1),
          "384x2": (384, 2, 8, 1, 1)}


def build(la, depth=4):
    st = build_stages(build_layers(bp.CONFIG1_DIMS, bp.CONFIG1_ACTS), depth, torch_init(0, dev), device=dev)
    launch = _lib.make_launch(*la) if la else None
    return st, [OptimizerState(OptimizerConfig("adam"), s.param_names, device=dev, launch=launch) for s in st]


graphs = {}
for name, la in shapes.items():
    for strategy in ("async_raw", "optimizer_prediction"):
        st, opts = build(la)
        g = GraphedExecute(build_timeline(strategy, 4, n), st, opts, strategy, data, "softmax_xent",
                           lambda mb: 1e-4, warmup_runs=1, streams="stage")
        g.replay()
        graphs[(name, strategy)] = (g, st, opts)
torch.cuda.synchronize()
times = {k: [] for k in graphs}
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _ in range(7):
    for k, (g, _, _) in graphs.items():
        e0.record()
        for _ in range(3):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        times[k].append(e0.elapsed_time(e1) / 3e3)
for name in shapes:
    off = n * bp.BATCH / statistics.median(times[(name, "async_raw")])
    on = n * bp.BATCH / statistics.median(times[(name, "optimizer_prediction")])
    print(json.dumps({"shared_gpu_run": name, "pred_off": round(off), "pred_on": round(on),
                      "overhead": round(1 - on / off, 4)}), flush=True)
del graphs
torch.cuda.empty_cache()
for name in ("default", "512x2", "256x4"):
    u = bp.stage_unit_times(torch, dev, lambda la=shapes[name]: build(la), data, "softmax_xent")
    print(json.dumps({"alone_units": name, "unit_us_off": [round(t * 1e6, 2) for t in u["pred_off"]],
                      "unit_us_on": [round(t * 1e6, 2) for t in u["pred_on"]]}), flush=True)
