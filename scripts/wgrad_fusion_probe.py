"""Config-1 single-GPU pipeline and per-stage unit times with the weight
gradients fused into the update (stages.FUSE_WGRAD_UPDATE, po_wgrad_update)
vs the split-K tensor-core GEMM + K2/K3. Graphed stage-concurrent runs,
prediction on/off, variants replayed in alternation.

  python scripts/wgrad_fusion_probe.py [--tf32]
"""
import argparse
import json
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2312_00839_b200 import bench_pipeline as bp  # noqa: E402
from paper_2312_00839_b200 import stages as S  # noqa: E402
from paper_2312_00839_b200.optim import OptimizerConfig, OptimizerState  # noqa: E402
from paper_2312_00839_b200.runtime import GraphedExecute, build_timeline  # noqa: E402
from paper_2312_00839_b200.stages import build_layers, build_stages, torch_init  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--tf32", action="store_true")
a = ap.parse_args()
torch.backends.cuda.matmul.allow_tf32 = a.tf32
dev = torch.device("cuda", 0)
data = bp.DeviceBatches(torch, dev)
graphs, finals = {}, {}
for fuse in (False, True):
    S.FUSE_WGRAD_UPDATE = fuse
    for strategy in ("async_raw", "optimizer_prediction"):
        st = build_stages(build_layers(bp.CONFIG1_DIMS, bp.CONFIG1_ACTS), 4, torch_init(0, dev), device=dev)
        opts = [OptimizerState(OptimizerConfig("adam"), s.param_names, device=dev) for s in st]
        g = GraphedExecute(build_timeline(strategy, 4, 64), st, opts, strategy, data, "softmax_xent",
                           lambda mb: 1e-4, streams="stage")
        g.replay()
        graphs[(fuse, strategy)] = (g, st)
S.FUSE_WGRAD_UPDATE = True
torch.cuda.synchronize()
times = {k: [] for k in graphs}
for _ in range(9):
    for k, (g, _) in graphs.items():
        times[k].append(bp._time_replays(torch, dev, g, 3))
for fuse in (False, True):
    off = 64 * bp.BATCH / statistics.median(times[(fuse, "async_raw")])
    on = 64 * bp.BATCH / statistics.median(times[(fuse, "optimizer_prediction")])
    print(json.dumps({"tf32": a.tf32, "fused_wgrad": fuse, "pred_off": round(off), "pred_on": round(on),
                      "overhead": round(1 - on / off, 4)}), flush=True)
# the runs trained the same model from the same init: losses agree within fp32 GEMM-order noise
la = graphs[(False, "optimizer_prediction")][0].report().losses
lb = graphs[(True, "optimizer_prediction")][0].report().losses
print(json.dumps({"final_loss_unfused": la[-1], "final_loss_fused": lb[-1]}), flush=True)
del graphs
torch.cuda.empty_cache()
for fuse in (False, True):
    S.FUSE_WGRAD_UPDATE = fuse

    def make():
        st = build_stages(build_layers(bp.CONFIG1_DIMS, bp.CONFIG1_ACTS), 4, torch_init(7, dev), device=dev)
        return st, [OptimizerState(OptimizerConfig("adam"), s.param_names, device=dev) for s in st]

    u = bp.stage_unit_times(torch, dev, make, data, "softmax_xent")
    print(json.dumps({"tf32": a.tf32, "fused_wgrad": fuse, "unit_off_us": [round(t * 1e6, 1) for t in u["pred_off"]],
                      "unit_on_us": [round(t * 1e6, 1) for t in u["pred_on"]]}), flush=True)
S.FUSE_WGRAD_UPDATE = True
