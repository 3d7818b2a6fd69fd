"""ncu driver: K2 and K3 (Adam) at a pipeline-stage size, buffers warm in L2
(run under ncu --cache-control none)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2312_00839_b200.optim import FlatParams, OptimizerConfig, OptimizerState  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 3146752
dev = torch.device("cuda", 0)
flat = FlatParams.from_tensors(["w"], [torch.randn(n) * 0.02], dev)
flat.grad.normal_(0, 1e-2)
staging = flat.layout.empty(dev)
opt = OptimizerState(OptimizerConfig("adam"), ["w"], device=dev, eager_checks=False)
for _ in range(3):
    opt.step_(flat, 1e-4)
    opt.step_predict_(flat, 1e-4, 1e-4, 3, staging)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
opt.step_(flat, 1e-4)
opt.step_predict_(flat, 1e-4, 1e-4, 3, staging)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
