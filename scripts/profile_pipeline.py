"""Driver for an ncu launch list of ONE CUDA-graph replay of a config-1 1F1B
run (prediction on or off), for the per-kernel time breakdown.

  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --cache-control none --clock-control none --csv --log-file gpurun_out/pipe_on.csv \
      python scripts/profile_pipeline.py --strategy optimizer_prediction
"""
import argparse
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2312_00839_b200.bench_pipeline import CONFIG1_ACTS, CONFIG1_DIMS, DeviceBatches  # noqa: E402
from paper_2312_00839_b200.optim import OptimizerConfig, OptimizerState  # noqa: E402
from paper_2312_00839_b200.runtime import GraphedExecute, build_timeline  # noqa: E402
from paper_2312_00839_b200.stages import build_layers, build_stages, torch_init  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--strategy", default="optimizer_prediction")
ap.add_argument("--n", type=int, default=16)
ap.add_argument("--tf32", action="store_true")
ap.add_argument("--streams", default="stage", choices=["stage", "serial"])
a = ap.parse_args()
torch.backends.cuda.matmul.allow_tf32 = a.tf32
dev = torch.device("cuda", 0)
data = DeviceBatches(torch, dev)
stages = build_stages(build_layers(CONFIG1_DIMS, CONFIG1_ACTS), 4, torch_init(0, dev), device=dev)
opts = [OptimizerState(OptimizerConfig("adam"), s.param_names, device=dev) for s in stages]
g = GraphedExecute(build_timeline(a.strategy, 4, a.n), stages, opts, a.strategy, data, "softmax_xent",
                   lambda mb: 1e-4, warmup_runs=1, streams=a.streams)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
g.replay()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("replayed", a.strategy, g.report().losses[-1])
