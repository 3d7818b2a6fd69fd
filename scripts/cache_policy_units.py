"""Optimizer cache policy vs per-stage unit times (one stage alone: the
one-stage-per-GPU setting) and vs the single-GPU stage-concurrent pipeline,
config 1, fp32 and TF32 GEMMs. cache: 1 streaming (.cs), 3 plain ld/st,
4 mixed (W, W_hat plain; G, state streaming)."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2312_00839_b200 import _lib  # noqa: E402
from paper_2312_00839_b200 import bench_pipeline as bp  # noqa: E402
from paper_2312_00839_b200.optim import OptimizerConfig, OptimizerState  # noqa: E402
from paper_2312_00839_b200.runtime import GraphedExecute, build_timeline  # noqa: E402
from paper_2312_00839_b200.stages import build_layers, build_stages, torch_init  # noqa: E402

dev = torch.device("cuda", 0)
data = bp.DeviceBatches(torch, dev)
dims, acts = bp.CONFIG1_DIMS, bp.CONFIG1_ACTS
for tf32 in (False, True):
    torch.backends.cuda.matmul.allow_tf32 = tf32
    for cache in (1, 3, 4):
        la = _lib.make_launch(0, 0, 0, cache, 0)

        def make():
            st = build_stages(build_layers(dims, acts), 4, torch_init(7, dev), device=dev)
            return st, [OptimizerState(OptimizerConfig("adam"), s.param_names, device=dev, launch=la) for s in st]

        u = bp.stage_unit_times(torch, dev, make, data, "softmax_xent")
        res = {}
        for strategy in ("async_raw", "optimizer_prediction"):
            st, opts = make()
            g = GraphedExecute(build_timeline(strategy, 4, 64), st, opts, strategy, data, "softmax_xent",
                               lambda mb: 1e-4, streams="stage")
            g.replay()
            torch.cuda.synchronize()
            res[strategy] = round(64 * bp.BATCH / bp._time_replays(torch, dev, g, 5))
            del g, st, opts
        print(json.dumps({"tf32": tf32, "cache": cache, "unit_off_us": [round(t * 1e6, 1) for t in u["pred_off"]],
                          "unit_on_us": [round(t * 1e6, 1) for t in u["pred_on"]], "pipe": res}), flush=True)
