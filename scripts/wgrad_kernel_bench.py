"""The fused weight-gradient + update kernel (po_wgrad_update) vs the split
tensor-core GEMM (po_gemm_f32x3, as stage_backward runs it) + K3 / K2, at the
config-1 stage shapes, CUDA-graph timed (20 back-to-back launches per replay,
L2-warm like a pipeline stage). Also the ncu driver: --ncu launches each form
a few times between cudaProfilerStart/Stop.

  python scripts/wgrad_kernel_bench.py [--ncu]
"""
import argparse
import ctypes
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2312_00839_b200 import _lib  # noqa: E402
from paper_2312_00839_b200.optim import OptimizerConfig  # noqa: E402
from paper_2312_00839_b200.stages import _weight_grad  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--ncu", action="store_true")
a = ap.parse_args()
lib = _lib.load()
dev = torch.device("cuda", 0)
hp = OptimizerConfig("adam").hparams()
H = ctypes.byref(hp)
for rows, fin, fout in ((128, 3072, 1024), (128, 1024, 1024)):
    g = torch.Generator(device=dev).manual_seed(0)
    x = torch.randn(rows, fin, device=dev, generator=g)
    dp = torch.randn(rows, fout, device=dev, generator=g) * 0.01
    w = torch.randn(fin, fout, device=dev, generator=g) * 0.02
    m = torch.zeros_like(w)
    v = torch.zeros_like(w)
    gw = torch.empty_like(w)
    wh = torch.empty_like(w)
    def cs():
        return torch.cuda.current_stream().cuda_stream

    def fused():
        _lib.check(lib.po_wgrad_update(H, x.data_ptr(), fin, dp.data_ptr(), fout, rows, fin, fout, w.data_ptr(),
                                       m.data_ptr(), v.data_ptr(), wh.data_ptr(), None, 1e-4, 3e-4, 5, None, None,
                                       0, cs()), "fused")

    def unfused():
        _weight_grad(x, dp, gw, False)
        _lib.check(lib.po_step_predict(H, w.data_ptr(), gw.data_ptr(), m.data_ptr(), v.data_ptr(), wh.data_ptr(),
                                       w.numel(), 1e-4, 3e-4, 5, None, None, cs()), "k3")

    def gemm_only():
        _weight_grad(x, dp, gw, False)

    def k3_only():
        _lib.check(lib.po_step_predict(H, w.data_ptr(), gw.data_ptr(), m.data_ptr(), v.data_ptr(), wh.data_ptr(),
                                       w.numel(), 1e-4, 3e-4, 5, None, None, cs()), "k3")

    forms = {"fused": fused, "gemm+k3": unfused, "gemm": gemm_only, "k3": k3_only}
    if a.ncu:
        for f in forms.values():
            f()
        torch.cuda.synchronize()
        torch.cuda.cudart().cudaProfilerStart()
        for f in forms.values():
            for _ in range(3):
                f()
        torch.cuda.synchronize()
        torch.cuda.cudart().cudaProfilerStop()
        continue
    res = {}
    for name, f in forms.items():
        for _ in range(3):
            f()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            for _ in range(20):
                f()
        graph.replay()
        torch.cuda.synchronize()
        ts = []
        for _ in range(7):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            graph.replay()
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3 / 20)
        res[name] = round(sorted(ts)[3], 2)
    print(json.dumps({"shape": [rows, fin, fout], "us": res}), flush=True)
