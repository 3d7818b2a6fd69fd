"""Config-1 graphed pipeline throughput under different optimizer launch
shapes / cache policies (small-N regime: 1M-3M-param stages)."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2312_00839_b200 import _lib  # noqa: E402
from paper_2312_00839_b200.bench_pipeline import BATCH, CONFIG1_ACTS, CONFIG1_DIMS, DeviceBatches  # noqa: E402
from paper_2312_00839_b200.optim import OptimizerConfig, OptimizerState  # noqa: E402
from paper_2312_00839_b200.runtime import GraphedExecute, build_timeline  # noqa: E402
from paper_2312_00839_b200.stages import build_layers, build_stages, torch_init  # noqa: E402

dev = torch.device("cuda", 0)
data = DeviceBatches(torch, dev)
n = 64
STREAMS = sys.argv[1] if len(sys.argv) > 1 else "stage"
variants = {"default": None}
for block, cps, unroll in ((128, 16, 1), (256, 8, 1), (128, 8, 1), (256, 4, 1), (512, 2, 1), (128, 4, 2)):
    for cache in (1, 4):
        variants[f"{block}x{cps}u{unroll}c{cache}"] = (block, cps, 8, cache, unroll)
for tf32 in (False,):
    torch.cuda.empty_cache()
    torch.backends.cuda.matmul.allow_tf32 = tf32
    for name, la in variants.items():
        res = {}
        for strategy in ("async_raw", "optimizer_prediction"):
            stages = build_stages(build_layers(CONFIG1_DIMS, CONFIG1_ACTS), 4, torch_init(0, dev), device=dev)
            launch = _lib.make_launch(*la) if la else None
            opts = [OptimizerState(OptimizerConfig("adam"), s.param_names, device=dev, launch=launch) for s in stages]
            g = GraphedExecute(build_timeline(strategy, 4, n), stages, opts, strategy, data, "softmax_xent",
                               lambda mb: 1e-4, warmup_runs=1, streams=STREAMS)
            g.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(5):
                g.replay()
            e1.record()
            torch.cuda.synchronize()
            res[strategy] = n * BATCH / (e0.elapsed_time(e1) / 5e3)
            del g, stages, opts
        on, off = res["optimizer_prediction"], res["async_raw"]
        print(json.dumps({"tf32": tf32, "variant": name, "pred_on": round(on), "pred_off": round(off),
                          "overhead": round(1 - on / off, 4)}), flush=True)
