"""Driver for an ncu capture of the fused DP kernel (po_dp_kernel) with one
replica (gloo world of 1): the streaming part's traffic must equal K3's."""
import os
import sys
from pathlib import Path

import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2312_00839_b200.dp_fused import FusedDPGroup  # noqa: E402
from paper_2312_00839_b200.optim import FlatLayout, FlatParams, OptimizerConfig, OptimizerState  # noqa: E402

os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29533")
dist.init_process_group("gloo", rank=0, world_size=1)
dev = torch.device("cuda", 0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 28
lay = FlatLayout(["w"], [(n,)])
grp = FusedDPGroup(dist, None, 0, 1, lay.numel, dev)
flat = FlatParams(lay, dev, torch.randn(lay.numel, device=dev) * 0.02)
opt = OptimizerState(OptimizerConfig("adam"), ["w"], device=dev)
out = torch.empty(lay.numel, device=dev)
for _ in range(4):
    grp.grad.normal_(0, 0.01)
    grp.step_predict(opt, flat, 1e-3, 1e-3, 3, out)
torch.cuda.synchronize()
grp.check()
dist.destroy_process_group()
print("done")
