"""Config-1 per-stage unit times (the one-stage-per-GPU projection's input,
16-unit graphs) under different small-N optimizer launch shapes
(block, CTAs/SM, unroll, cache) for every K2/K3 of the unit.

  python scripts/unit_shape_probe.py [--default-only]
"""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2312_00839_b200 import _lib  # noqa: E402
from paper_2312_00839_b200 import bench_pipeline as bp  # noqa: E402
from paper_2312_00839_b200.optim import OptimizerConfig, OptimizerState  # noqa: E402
from paper_2312_00839_b200.stages import build_layers, build_stages, torch_init  # noqa: E402

torch.backends.cuda.matmul.allow_tf32 = False
dev = torch.device("cuda", 0)
data = bp.DeviceBatches(torch, dev)
shapes = [(0, 0, 0, 0), (128, 16, 1, 1), (128, 8, 1, 1), (256, 8, 1, 1), (256, 4, 1, 1), (512, 4, 1, 1),
          (512, 2, 1, 1), (512, 1, 1, 1), (128, 16, 1, 3), (256, 8, 3, 1)]
if "--default-only" in sys.argv:  # repeat the default shape: the measurement's own spread
    shapes = [(0, 0, 0, 0)] * 4
for sh in shapes:
    la = None if sh == (0, 0, 0, 0) else _lib.make_launch(sh[0], sh[1], 8, sh[3], sh[2])

    def make(la=la):
        st = build_stages(build_layers(bp.CONFIG1_DIMS, bp.CONFIG1_ACTS), 4, torch_init(7, dev), device=dev)
        return st, [OptimizerState(OptimizerConfig("adam"), s.param_names, device=dev, launch=la) for s in st]

    u = bp.stage_unit_times(torch, dev, make, data, "softmax_xent", reps=5)
    off, on = u["pred_off"], u["pred_on"]
    print(json.dumps({"shape": "default" if sh == (0, 0, 0, 0) else list(sh),
                      "off_us": [round(t * 1e6, 2) for t in off], "on_us": [round(t * 1e6, 2) for t in on],
                      "bottleneck_overhead": round(1 - max(off) / max(on), 4)}), flush=True)
