"""Where does stage 0's prediction cost go? Config-1 stage-0 unit graph
(forward + backward + update) timed with: K2 (prediction off), K3 (on),
K3 but the forward reading the live weights, K2 + a plain copy W -> staging,
and the update alone (K2 / K3)."""
import json
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2312_00839_b200 import bench_pipeline as bp  # noqa: E402
from paper_2312_00839_b200.optim import OptimizerConfig, OptimizerState  # noqa: E402
from paper_2312_00839_b200.stages import build_layers, build_stages, torch_init  # noqa: E402

torch.backends.cuda.matmul.allow_tf32 = "--tf32" in sys.argv
dev = torch.device("cuda", 0)
data = bp.DeviceBatches(torch, dev)
x0, y0 = data.batch(1)
g_last = torch.randn(128, 1024, device=dev)


def make(variant):
    st = build_stages(build_layers(bp.CONFIG1_DIMS, bp.CONFIG1_ACTS), 4, torch_init(7, dev), device=dev)[0]
    opt = OptimizerState(OptimizerConfig("adam"), st.param_names, device=dev)
    staging = st.flat.layout.empty(dev)
    sviews = st.flat.layout.views(staging)
    opt._bind(st.flat.layout)
    opt._ensure_state()
    opt.eager_checks = False

    def unit():
        if variant.startswith("opt_"):
            (opt.step_predict_(st.flat, 1e-4, 1e-4, 3, staging) if variant == "opt_k3" else opt.step_(st.flat, 1e-4))
            return
        w = sviews if variant in ("k3", "k2_copy") else st.params
        st.run_forward(w, (0, 0), x0, 1, check_finite=False)
        st.run_backward(st.params, (0, 0), g_last, need_input_grad=False)
        if variant in ("k3", "k3_fwd_live"):
            opt.step_predict_(st.flat, 1e-4, 1e-4, 3, staging)
        else:
            opt.step_(st.flat, 1e-4)
            if variant == "k2_copy":
                staging.copy_(st.flat.data)

    for _ in range(2):
        unit()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=torch.cuda.Stream() if "--fresh" in sys.argv else None):
        unit()
    g.replay()
    torch.cuda.synchronize()
    g.keepalive = (opt, staging, sviews)  # the graph replays into their memory
    return g, st


variants = sys.argv[sys.argv.index("--v") + 1].split(",") if "--v" in sys.argv else ["k2", "k3", "k3_fwd_live", "k2_copy", "opt_k2", "opt_k3"]
graphs = {v: make(v) for v in variants}
times = {v: [] for v in variants}
for _ in range(7):
    for v, (g, _) in graphs.items():
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        times[v].append(e0.elapsed_time(e1) * 1e3 / 20)
print(json.dumps({v: round(statistics.median(t), 2) for v, t in times.items()}))
for v, (g, st) in graphs.items():
    print(v, "finite W", bool(torch.isfinite(st.flat.data).all()), "finite G", bool(torch.isfinite(st.flat.grad).all()),
          "numel", st.flat.layout.numel)
