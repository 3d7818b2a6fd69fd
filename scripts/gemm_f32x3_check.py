"""po_gemm_f32x3 (tcgen05 fast-FP32 GEMM) vs float64 and vs the SIMT fp32
GEMMs the stage math used, on the config-1 shapes: forward (x @ W, split-K),
weight gradient (x^T @ dpre) and input gradient (dpre @ W^T, split-K).
Accuracy and CUDA-graph timing."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2312_00839_b200 import _lib  # noqa: E402

torch.backends.cuda.matmul.allow_tf32 = False
dev = torch.device("cuda", 0)
lib = _lib.load()
cs = lambda: torch.cuda.current_stream().cuda_stream  # noqa: E731


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


def report(name, ours, simt, got, ref):
    ours()
    torch.cuda.synchronize()
    r = ref()
    err = float((got().double() - r).abs().max() / r.abs().max())
    print(json.dumps({"case": name, "us_f32x3": round(t_graph(ours), 2), "us_simt": round(t_graph(simt), 2),
                      "relerr_f32x3": err}), flush=True)


B = 128
for din, dout in ((3072, 1024), (1024, 1024)):
    x = torch.randn(B, din, device=dev)
    w = torch.randn(din, dout, device=dev) / din ** 0.5
    dpre = torch.randn(B, dout, device=dev)
    for s in (1, 2, 4, 8):  # forward, split-K over din
        ks = din // s
        out = torch.empty(s, B, dout, device=dev)

        def fwd(s=s, ks=ks, out=out):
            assert lib.po_gemm_f32x3(0, 0, x.data_ptr(), din, ks, w.data_ptr(), dout, ks * dout, out.data_ptr(), B,
                                     dout, ks, s, None, 0, cs()) == 0

        report(f"fwd {din}x{dout} S{s}", fwd,
               lambda s=s, ks=ks: torch.bmm(x.view(B, s, ks).transpose(0, 1), w.view(s, ks, dout)),
               lambda out=out: out.sum(0), lambda: x.double() @ w.double())
    gw = torch.empty(din, dout, device=dev)

    def wgrad():
        assert lib.po_gemm_f32x3(1, 0, x.data_ptr(), din, 0, dpre.data_ptr(), dout, 0, gw.data_ptr(), din, dout, B, 1,
                                 None, 0, cs()) == 0

    report(f"wgrad {din}x{dout}", wgrad, lambda: torch.mm(x.t(), dpre), lambda: gw,
           lambda: x.double().t() @ dpre.double())
    for s in (1, 2, 4, 8):  # input gradient, split-K over dout
        ks = dout // s
        gi = torch.empty(s, B, din, device=dev)

        def dgrad(s=s, ks=ks, gi=gi):
            assert lib.po_gemm_f32x3(0, 1, dpre.data_ptr(), dout, ks, w.data_ptr(), dout, ks, gi.data_ptr(), B, din,
                                     ks, s, None, 0, cs()) == 0

        report(f"dgrad {din}x{dout} S{s}", dgrad, lambda: torch.mm(dpre, w.t()), lambda gi=gi: gi.sum(0),
               lambda: dpre.double() @ w.double().t())
