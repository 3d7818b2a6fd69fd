"""Config-1 stage-concurrent graphed pipeline with CUDA stream priorities on
the stage lanes (runtime.LANE_PRIORITY): does giving the bottleneck stage's
kernels priority raise throughput? Prediction on/off, variants replayed in
alternation (median of 9)."""
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

lo, hi = torch.cuda.Stream.priority_range() if hasattr(torch.cuda.Stream, "priority_range") else (0, -1)
print(json.dumps({"priority_range": [lo, hi]}), flush=True)
variants = {"none": {}, "stage0": {0: -1}, "last": {3: -1}, "rev_ramp2": {3: -2, 2: -1}, "rev_ramp3": {3: -3, 2: -2, 1: -1}, "last_two": {3: -1, 2: -1}}
dev = torch.device("cuda", 0)
data = bp.DeviceBatches(torch, dev)
graphs = {}
for name, prio in variants.items():
    runtime.LANE_PRIORITY = prio
    for strategy in ("async_raw", "optimizer_prediction"):
        st = build_stages(build_layers(bp.CONFIG1_DIMS, bp.CONFIG1_ACTS), 4, torch_init(0, dev), device=dev)
        opts = [OptimizerState(OptimizerConfig("adam"), s.param_names, device=dev) for s in st]
        g = GraphedExecute(build_timeline(strategy, 4, 64), st, opts, strategy, data, "softmax_xent",
                           lambda mb: 1e-4, streams="stage")
        g.replay()
        graphs[(name, strategy)] = g
runtime.LANE_PRIORITY = {}
torch.cuda.synchronize()
times = {k: [] for k in graphs}
for _ in range(9):
    for k, g in graphs.items():
        times[k].append(bp._time_replays(torch, dev, g, 3))
for name in variants:
    off = 64 * bp.BATCH / statistics.median(times[(name, "async_raw")])
    on = 64 * bp.BATCH / statistics.median(times[(name, "optimizer_prediction")])
    print(json.dumps({"variant": name, "priorities": variants[name], "pred_off": round(off), "pred_on": round(on),
                      "overhead": round(1 - on / off, 4)}), flush=True)
