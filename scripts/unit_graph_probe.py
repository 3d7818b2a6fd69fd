"""Per-stage unit times of config 1 measured with 1 unit per CUDA graph
(every unit pays a graph launch gap) vs 16 back-to-back units per graph
(the stage's steady state on its own GPU), twice each: the projection's
noise and bias."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2312_00839_b200 import bench_pipeline as bp  # noqa: E402
from paper_2312_00839_b200.optim import OptimizerConfig, OptimizerState  # noqa: E402
from paper_2312_00839_b200.stages import build_layers, build_stages, torch_init  # noqa: E402

torch.backends.cuda.matmul.allow_tf32 = False
dev = torch.device("cuda", 0)
data = bp.DeviceBatches(torch, dev)


def make():
    st = build_stages(build_layers(bp.CONFIG1_DIMS, bp.CONFIG1_ACTS), 4, torch_init(7, dev), device=dev)
    return st, [OptimizerState(OptimizerConfig("adam"), s.param_names, device=dev) for s in st]


for units, reps in ((1, 40), (16, 5), (1, 40), (16, 5)):
    u = bp.stage_unit_times(torch, dev, make, data, "softmax_xent", reps=reps, units=units)
    off, on = u["pred_off"], u["pred_on"]
    print(json.dumps({"units_per_graph": units, "off_us": [round(t * 1e6, 2) for t in off],
                      "on_us": [round(t * 1e6, 2) for t in on],
                      "bottleneck_overhead": round(1 - max(off) / max(on), 4)}), flush=True)
