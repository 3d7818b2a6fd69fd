"""Config-1 stage-concurrent graphed pipeline (the bench headline setting)
under different small-N optimizer launch shapes: every K1/K2/K3 of the run
takes the given (block, CTAs/SM, unroll, cache); prediction on/off, all
variants' graphs replayed in alternation (median of trials).

  python scripts/small_shape_pipeline.py [--tf32]
"""
import argparse
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

ap = argparse.ArgumentParser()
ap.add_argument("--tf32", action="store_true")
ap.add_argument("--shapes", default="0,0,0,0;128,16,1,1;128,8,1,1;256,4,1,1;256,2,1,1;512,1,1,1;512,2,1,1;"
                                    "64,16,1,1;128,4,1,1;128,8,3,1;256,2,3,1")
ap.add_argument("--trials", type=int, default=7)
a = ap.parse_args()
torch.backends.cuda.matmul.allow_tf32 = a.tf32
dev = torch.device("cuda", 0)
data = bp.DeviceBatches(torch, dev)
graphs = {}
shapes = [tuple(int(x) for x in s.split(",")) for s in a.shapes.split(";")]
for sh in shapes:
    la = None if sh == (0, 0, 0, 0) else _lib.make_launch(sh[0], sh[1], 8, sh[3], sh[2])
    for strategy in ("async_raw", "optimizer_prediction"):
        st = build_stages(build_layers(bp.CONFIG1_DIMS, bp.CONFIG1_ACTS), 4, torch_init(0, dev), device=dev)
        opts = [OptimizerState(OptimizerConfig("adam"), s.param_names, device=dev, launch=la) for s in st]
        g = GraphedExecute(build_timeline(strategy, 4, 64), st, opts, strategy, data, "softmax_xent",
                           lambda mb: 1e-4, streams="stage")
        g.replay()
        graphs[(sh, strategy)] = g
torch.cuda.synchronize()
times = {k: [] for k in graphs}
for _ in range(a.trials):
    for k, g in graphs.items():
        times[k].append(bp._time_replays(torch, dev, g, 3))
for sh in shapes:
    off = 64 * bp.BATCH / statistics.median(times[(sh, "async_raw")])
    on = 64 * bp.BATCH / statistics.median(times[(sh, "optimizer_prediction")])
    print(json.dumps({"tf32": a.tf32, "shape": "default" if sh == (0, 0, 0, 0) else list(sh), "pred_off": round(off),
                      "pred_on": round(on), "overhead": round(1 - on / off, 4)}), flush=True)
