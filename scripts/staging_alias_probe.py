"""Config-1 stage-concurrent graphed pipeline with W_hat in a separate
staging buffer vs in the gradient's storage (runtime.STAGING_IN_GRAD),
prediction on/off, fp32 and TF32 GEMMs, graphs replayed in alternation.

  python scripts/staging_alias_probe.py
"""
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
    for alias in (False, True):
        runtime.STAGING_IN_GRAD = alias
        for strategy in ("async_raw", "optimizer_prediction"):
            st = build_stages(build_layers(bp.CONFIG1_DIMS, bp.CONFIG1_ACTS), 4, torch_init(0, dev), device=dev)
            opts = [OptimizerState(OptimizerConfig("adam"), s.param_names, device=dev) for s in st]
            g = GraphedExecute(build_timeline(strategy, 4, 64), st, opts, strategy, data, "softmax_xent",
                               lambda mb: 1e-4, streams="stage")
            g.replay()
            graphs[(alias, strategy)] = (g, st)
    runtime.STAGING_IN_GRAD = True
    torch.cuda.synchronize()
    times = {k: [] for k in graphs}
    for _ in range(9):
        for k, (g, _) in graphs.items():
            times[k].append(bp._time_replays(torch, dev, g, 3))
    same = all(torch.equal(a, b) for a, b in zip(
        [p for s in graphs[(False, "optimizer_prediction")][1] for p in s.params],
        [p for s in graphs[(True, "optimizer_prediction")][1] for p in s.params]))
    for alias in (False, True):
        off = 64 * bp.BATCH / statistics.median(times[(alias, "async_raw")])
        on = 64 * bp.BATCH / statistics.median(times[(alias, "optimizer_prediction")])
        print(json.dumps({"tf32": tf32, "staging_in_grad": alias, "pred_off": round(off), "pred_on": round(on),
                          "overhead": round(1 - on / off, 4), "weights_bit_identical": same}), flush=True)
    del graphs
    torch.cuda.empty_cache()
