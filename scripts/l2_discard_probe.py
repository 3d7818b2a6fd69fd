"""Config-1 pipeline with dead-buffer L2 discards (runtime.L2_DISCARD): the
staging buffer after each predicted forward, the gradient after each update.
Graphed stage-concurrent runs, prediction on/off, variants in alternation."""
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

dev = torch.device("cuda", 0)
for tf32 in (False, True):
    torch.backends.cuda.matmul.allow_tf32 = tf32
    data = bp.DeviceBatches(torch, dev)
    graphs = {}
    for variant in ("none", "staging", "grad", "both"):
        runtime.L2_DISCARD.update(staging=variant in ("staging", "both"), grad=variant in ("grad", "both"))
        for strategy in ("async_raw", "optimizer_prediction"):
            st = build_stages(build_layers(bp.CONFIG1_DIMS, bp.CONFIG1_ACTS), 4, torch_init(0, dev), device=dev)
            opts = [OptimizerState(OptimizerConfig("adam"), s.param_names, device=dev) for s in st]
            g = GraphedExecute(build_timeline(strategy, 4, 64), st, opts, strategy, data, "softmax_xent",
                               lambda mb: 1e-4, streams="stage")
            g.replay()
            graphs[(variant, strategy)] = g
    runtime.L2_DISCARD.update(staging=False, grad=False)
    torch.cuda.synchronize()
    times = {k: [] for k in graphs}
    for _ in range(7):
        for k, g in graphs.items():
            times[k].append(bp._time_replays(torch, dev, g, 3))
    for variant in ("none", "staging", "grad", "both"):
        off = 64 * bp.BATCH / statistics.median(times[(variant, "async_raw")])
        on = 64 * bp.BATCH / statistics.median(times[(variant, "optimizer_prediction")])
        print(json.dumps({"tf32": tf32, "variant": variant, "pred_off": round(off), "pred_on": round(on),
                          "overhead": round(1 - on / off, 4)}), flush=True)
    del graphs
    torch.cuda.empty_cache()
