"""torch.profiler kernel breakdown of one module stage's unit (forward +
backward + K2) for configs 2-4 (which stage, dtype and layout selectable)."""
import argparse
import sys
from pathlib import Path

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2312_00839_b200 import bench_pipeline as bp  # noqa: E402
from paper_2312_00839_b200.optim import OptimizerConfig, OptimizerState  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="config3_resnet101")
ap.add_argument("--stage", type=int, default=4)
ap.add_argument("--amp", default=None)
ap.add_argument("--top", type=int, default=25)
ap.add_argument("--cudnn-bn", action="store_true", help="put cuDNN batch norm back (single-stream use only)")
a = ap.parse_args()
torch.backends.cudnn.allow_tf32 = torch.backends.cuda.matmul.allow_tf32 = True
dev = torch.device("cuda", 0)
cfg = bp.MODULE_CONFIGS[a.config]
stages, _ = bp.module_stages_for(torch, a.config, dev, amp=a.amp)
st = stages[a.stage]
if a.cudnn_bn:
    from paper_2312_00839_b200.stage_models import use_cudnn_bn

    use_cudnn_bn([st])
opt = OptimizerState(OptimizerConfig(cfg["opt"]), st.param_names, device=dev, eager_checks=False)
data = bp.ModuleBatches(torch, dev, cfg)
x = data.batch(1)[0] if a.stage == 0 else torch.randn((cfg["batch"], *st.in_shape), device=dev)
g = torch.randn((cfg["batch"], *st.out_shape), device=dev)


def unit():
    st.run_forward(st.params, (0, 0), x, 1, check_finite=False)
    st.run_backward(st.params, (0, 0), g, need_input_grad=a.stage > 0)
    opt.step_(st.flat, 1e-3)


for _ in range(3):
    unit()
torch.cuda.synchronize()
from paper_2312_00839_b200.runtime import capture  # noqa: E402

graph = torch.cuda.CUDAGraph()
with capture(graph):
    unit()
graph.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    graph.replay()
e1.record()
torch.cuda.synchronize()
print(f"graphed unit: {e0.elapsed_time(e1) / 5:.3f} ms")
with profile(activities=[ProfilerActivity.CUDA]) as p:
    for _ in range(3):
        unit()
    torch.cuda.synchronize()
print(p.key_averages().table(sort_by="cuda_time_total", row_limit=a.top, max_name_column_width=90))
