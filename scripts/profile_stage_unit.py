"""ncu driver: replay the config-1 stage-k unit graph (forward + backward +
K2 or K3) a few times, prediction off then on, between cudaProfilerStart/Stop.

  ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --cache-control none --clock-control none --csv --log-file gpurun_out/unit.csv \
      python scripts/profile_stage_unit.py --stage 0
"""
import argparse
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2312_00839_b200 import bench_pipeline as bp  # noqa: E402
from paper_2312_00839_b200.optim import OptimizerConfig, OptimizerState  # noqa: E402
from paper_2312_00839_b200.stages import build_layers, build_stages, torch_init  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--stage", type=int, default=0)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--fuse-wgrad", action="store_true", help="stages.FUSE_WGRAD_UPDATE on (po_wgrad_update)")
a = ap.parse_args()
if a.fuse_wgrad:
    from paper_2312_00839_b200 import stages as _S

    _S.FUSE_WGRAD_UPDATE = True
torch.backends.cuda.matmul.allow_tf32 = False
dev = torch.device("cuda", 0)
data = bp.DeviceBatches(torch, dev)
graphs = {}
for key in ("pred_off", "pred_on"):
    st = build_stages(build_layers(bp.CONFIG1_DIMS, bp.CONFIG1_ACTS), 4, torch_init(7, dev), device=dev)
    opts = [OptimizerState(OptimizerConfig("adam"), s.param_names, device=dev) for s in st]
    graphs[key] = (bp._unit_graph(torch, dev, a.stage, st[a.stage], opts[a.stage], data, "softmax_xent",
                                  key == "pred_on", 4), st)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
for key in ("pred_off", "pred_on"):
    for _ in range(a.reps):
        graphs[key][0].replay()
    torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
