"""Config-1 graphed single-GPU pipeline (stages concurrent, one stream per
stage) with the tensor-core GEMMs' split-K count capped at 8 (default), 4
and 2: fewer K slices = fewer CTAs per GEMM (less SM time each, longer
latency), which may let concurrent stages' GEMMs share the GPU. Arms timed
in alternation, median of 5."""
import json
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2312_00839_b200 import stages as S  # noqa: E402
from paper_2312_00839_b200.bench_pipeline import BATCH, CONFIG1_ACTS, CONFIG1_DIMS, DeviceBatches  # noqa: E402
from paper_2312_00839_b200.optim import OptimizerConfig, OptimizerState  # noqa: E402
from paper_2312_00839_b200.runtime import GraphedExecute, build_timeline  # noqa: E402
from paper_2312_00839_b200.stages import build_layers, build_stages, torch_init  # noqa: E402

torch.backends.cuda.matmul.allow_tf32 = False
dev = torch.device("cuda", 0)
data = DeviceBatches(torch, dev)
n = 64
CAPS = tuple(int(c) for c in (sys.argv[2] if len(sys.argv) > 2 else "8,16,4").split(","))
STREAMS = sys.argv[1] if len(sys.argv) > 1 else "stage"
orig = S._splitk_tc


def capped(cap):
    """_splitk_tc with the slice count capped at `cap` (16: slices >= 128 up to 16)."""
    def f(rows, k):
        if rows > 512 or k < 256:
            return 1
        s = 1
        while s < cap and k % (s * 2) == 0 and k // (s * 2) >= 128:
            s *= 2
        return s
    return f


import os  # noqa: E402

from paper_2312_00839_b200 import _lib  # noqa: E402

PDL = os.environ.get("PDL") == "1"  # short stream kernels with programmatic dependent launch
graphs = {}
for cap in CAPS:
    S._splitk_tc = capped(cap)
    for strategy in ("async_raw", "optimizer_prediction"):
        stages = build_stages(build_layers(CONFIG1_DIMS, CONFIG1_ACTS), 4, torch_init(0, dev), device=dev)
        opts = [OptimizerState(OptimizerConfig("adam"), s.param_names, device=dev) for s in stages]
        with _lib.pdl(PDL):
            g = GraphedExecute(build_timeline(strategy, 4, n), stages, opts, strategy, data, "softmax_xent",
                               lambda mb: 1e-4, warmup_runs=1, streams=STREAMS)
        g.replay()
        graphs[(cap, strategy)] = (g, stages, opts)
S._splitk_tc = orig
torch.cuda.synchronize()
times = {k: [] for k in graphs}
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _ in range(5):
    for k, (g, _, _) in graphs.items():
        e0.record()
        for _ in range(5):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        times[k].append(e0.elapsed_time(e1) / 5e3)
for cap in CAPS:
    off = n * BATCH / statistics.median(times[(cap, "async_raw")])
    on = n * BATCH / statistics.median(times[(cap, "optimizer_prediction")])
    print(json.dumps({"streams": STREAMS, "pdl_short_kernels": PDL, "splitk_cap": cap, "pred_off": round(off), "pred_on": round(on),
                      "overhead": round(1 - on / off, 4)}), flush=True)
