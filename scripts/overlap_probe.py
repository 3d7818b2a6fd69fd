"""Can stage 0's update (K3) hide behind its next forward GEMM? Sequential
K3 -> split-K tensor-core GEMM vs K3 in 8 weight slices on one stream with
each GEMM K-slice on a second stream as soon as its W_hat slice is written."""
import ctypes
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2312_00839_b200 import _lib  # noqa: E402
from paper_2312_00839_b200.optim import OptimizerConfig  # noqa: E402

dev = torch.device("cuda", 0)
lib = _lib.load()
K, N, B, S = 3072, 1024, 128, 8
ks = K // S
w = torch.randn(K * N, device=dev) * 0.02
g = torch.randn(K * N, device=dev) * 1e-2
m = torch.zeros(K * N, device=dev)
v = torch.zeros(K * N, device=dev)
wh = torch.empty(K * N, device=dev)
x = torch.randn(B, K, device=dev)
part = torch.empty(S, B, N, device=dev)
bad = torch.full((1,), 2 ** 63 - 1, dtype=torch.int64, device=dev)
hp = OptimizerConfig("adam").hparams()
side = torch.cuda.Stream()


def k3(lo, n, stream):
    rc = lib.po_step_predict(ctypes.byref(hp), w.data_ptr() + 4 * lo, g.data_ptr() + 4 * lo, m.data_ptr() + 4 * lo,
                             v.data_ptr() + 4 * lo, wh.data_ptr() + 4 * lo, n, 1e-4, 3e-4, 5, bad.data_ptr(), None,
                             stream)
    assert rc == 0


def k2(lo, n, stream):
    rc = lib.po_step(ctypes.byref(hp), w.data_ptr() + 4 * lo, g.data_ptr() + 4 * lo, m.data_ptr() + 4 * lo,
                     v.data_ptr() + 4 * lo, None, n, 1e-4, 5, bad.data_ptr(), None, stream)
    assert rc == 0


def gemm(l0, nb, src, stream):
    rc = lib.po_gemm_f32x3(0, 0, x.data_ptr() + 4 * l0 * ks, K, ks, src.data_ptr() + 4 * l0 * ks * N, N, ks * N,
                           part.data_ptr() + 4 * l0 * B * N, B, N, ks, nb, None, 0, stream)
    assert rc == 0


def seq(upd, src):
    cs = torch.cuda.current_stream().cuda_stream
    upd(0, K * N, cs)
    gemm(0, S, src, cs)


def inter(upd, src):
    cur = torch.cuda.current_stream()
    side.wait_stream(cur)
    evs = []
    for l in range(S):
        upd(l * ks * N, ks * N, cur.cuda_stream)
        ev = torch.cuda.Event()
        ev.record(cur)
        evs.append(ev)
    for l in range(S):
        side.wait_event(evs[l])
        gemm(l, 1, src, side.cuda_stream)
    cur.wait_stream(side)


def t_graph(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        for _ in range(reps):
            fn()
    gr.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        gr.replay()
    e1.record()
    torch.cuda.synchronize()
    return round(e0.elapsed_time(e1) * 1e3 / (5 * reps), 2)


print(json.dumps({
    "k3_alone": t_graph(lambda: k3(0, K * N, torch.cuda.current_stream().cuda_stream)),
    "k2_alone": t_graph(lambda: k2(0, K * N, torch.cuda.current_stream().cuda_stream)),
    "gemm_alone": t_graph(lambda: gemm(0, S, wh, torch.cuda.current_stream().cuda_stream)),
    "seq_k3_gemm": t_graph(lambda: seq(k3, wh)),
    "seq_k2_gemm": t_graph(lambda: seq(k2, w)),
    "inter_k3_gemm": t_graph(lambda: inter(k3, wh)),
    "inter_k2_gemm": t_graph(lambda: inter(k2, w)),
}))
