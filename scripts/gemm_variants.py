"""Config-1 fp32 GEMM formulations (TF32 off): time each shape/layout variant
in a CUDA graph (launch overhead excluded), to pick the stage math's calls."""
import json

import torch

torch.backends.cuda.matmul.allow_tf32 = False
dev = torch.device("cuda", 0)


def t_graph(fn, reps=50):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / (5 * reps)


B = 128
for din, dout in ((3072, 1024), (1024, 1024), (1024, 10)):
    x = torch.randn(B, din, device=dev)
    w = torch.randn(din, dout, device=dev) * 0.02
    wt = w.t().contiguous()
    b = torch.randn(dout, device=dev)
    g = torch.randn(B, dout, device=dev)
    gw = torch.empty(din, dout, device=dev)
    gwt = torch.empty(dout, din, device=dev)
    out = torch.empty(B, dout, device=dev)
    gx = torch.empty(B, din, device=dev)
    fl = 2 * B * din * dout / 1e6
    res = {
        "fwd addmm_act (x@w, w row-major)": t_graph(lambda: torch._addmm_activation(b, x, w)),
        "fwd addmm_act (x@wt.T)": t_graph(lambda: torch._addmm_activation(b, x, wt.t())),
        "fwd mm only": t_graph(lambda: torch.mm(x, w, out=out)),
        "wgrad mm(x.T, g)": t_graph(lambda: torch.mm(x.t(), g, out=gw)),
        "wgrad mm(g.T, x) -> (dout,din)": t_graph(lambda: torch.mm(g.t(), x, out=gwt)),
        "wgrad mm(x.T.contig, g)": t_graph(lambda: torch.mm(x.t().contiguous(), g, out=gw)),
        "dgrad mm(g, w.T)": t_graph(lambda: torch.mm(g, w.t(), out=gx)),
        "dgrad mm(g, wt)": t_graph(lambda: torch.mm(g, wt, out=gx)),
    }
    print(json.dumps({"shape": [B, din, dout], "mflop": fl,
                      "us": {k: round(v, 2) for k, v in res.items()},
                      "tflops": {k: round(fl / v / 1e6 * 1e6 / 1e6, 1) for k, v in res.items()}}), flush=True)
