"""Programmatic dependent launch of the short stream kernels (po_set_pdl)
where a stage's work is alone on the GPU: config-1 per-stage unit times
(16 back-to-back units per graph, both modes) and the serial-stream /
D = 1 graphed runs, PDL off vs on (captured under each setting, replayed in
alternation). Also checks that PDL leaves the results bit-identical."""
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

torch.backends.cuda.matmul.allow_tf32 = False
dev = torch.device("cuda", 0)
data = bp.DeviceBatches(torch, dev)


def make():
    st = build_stages(build_layers(bp.CONFIG1_DIMS, bp.CONFIG1_ACTS), 4, torch_init(0, dev), device=dev)
    return st, [OptimizerState(OptimizerConfig("adam"), s.param_names, device=dev) for s in st]


for on in (False, True, False, True):
    with _lib.pdl(on):
        u = bp.stage_unit_times(torch, dev, make, data, "softmax_xent")
    print(json.dumps({"pdl": on, "unit_us_off": [round(t * 1e6, 2) for t in u["pred_off"]],
                      "unit_us_on": [round(t * 1e6, 2) for t in u["pred_on"]]}), flush=True)

n = 64
graphs, finals = {}, {}
for streams, depth in (("serial", 4), ("stage", 1)):
    for on in (False, True):
        for strategy in ("async_raw", "optimizer_prediction"):
            with _lib.pdl(on):
                st = build_stages(build_layers(bp.CONFIG1_DIMS, bp.CONFIG1_ACTS), depth, torch_init(0, dev), device=dev)
                opts = [OptimizerState(OptimizerConfig("adam"), s.param_names, device=dev) for s in st]
                g = GraphedExecute(build_timeline(strategy, depth, n), st, opts, strategy, data, "softmax_xent",
                                   lambda mb: 1e-4, warmup_runs=1, streams=streams)
            g.replay()
            torch.cuda.synchronize()
            graphs[(streams, depth, on, strategy)] = g
            finals[(streams, depth, on, strategy)] = [s.flat.data.clone() for s in st]
times = {k: [] for k in graphs}
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _ in range(5):
    for k, g in graphs.items():
        e0.record()
        for _ in range(3):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        times[k].append(e0.elapsed_time(e1) / 3e3)
for streams, depth in (("serial", 4), ("stage", 1)):
    for strategy in ("async_raw", "optimizer_prediction"):
        same = all(torch.equal(a, b) for a, b in zip(finals[(streams, depth, False, strategy)],
                                                     finals[(streams, depth, True, strategy)]))
        row = {"streams": streams, "depth": depth, "strategy": strategy, "bit_identical": same}
        for on in (False, True):
            row["pdl_on" if on else "pdl_off"] = round(n * bp.BATCH / statistics.median(times[(streams, depth, on,
                                                                                                  strategy)]))
        print(json.dumps(row), flush=True)
