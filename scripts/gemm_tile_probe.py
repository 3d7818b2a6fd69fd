"""po_gemm_f32x3 tile-shape variants (scripts/build_gemm_tile_variants.sh;
128 x N x K tiles, N <= 128 in this CUTLASS) on config 1's stage shapes:
forward x.W (split-K S), weight gradient x^T.dpre and input gradient
dpre.W^T (split-K S). CUDA-graph timing, 16 calls per graph, best of 5."""
import ctypes
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent))
from presplit_gemm_probe import t_graph  # noqa: E402  (module body is guarded below)

dev = torch.device("cuda", 0)
cs = lambda: torch.cuda.current_stream().cuda_stream  # noqa: E731
libs = {}
SMEM = {}
for p in sorted((Path(__file__).resolve().parent / "_probe_libs").glob("libgemm_*.so")):
    lib = ctypes.CDLL(str(p))
    f = lib.po_gemm_f32x3
    f.restype = ctypes.c_int
    f.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p,
                  ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                  ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p]
    libs[p.stem.replace("libgemm_", "")] = f
    try:
        lib.po_probe_gemm_smem.restype = ctypes.c_int
        SMEM[p.stem.replace("libgemm_", "")] = [lib.po_probe_gemm_smem(v) for v in range(3)]
    except AttributeError:
        pass

def t_conc(fn, streams=4, reps=16):
    """Per-GEMM time with `streams` streams each running `reps` of it
    concurrently inside one CUDA graph (the stage-concurrent runner's mix)."""
    ss = [torch.cuda.Stream() for _ in range(streams)]
    g = torch.cuda.CUDAGraph()
    fn()
    torch.cuda.synchronize()
    with torch.cuda.graph(g):
        cur = torch.cuda.current_stream()
        for st in ss:
            st.wait_stream(cur)
        for st in ss:
            with torch.cuda.stream(st):
                for _ in range(reps):
                    assert fn() == 0
        for st in ss:
            cur.wait_stream(st)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(5):
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e3 / (streams * reps))
    return round(best, 2)


B = 128
for din, dout in ((3072, 1024), (1024, 1024)):
    x = torch.randn(B, din, device=dev)
    w = torch.randn(din, dout, device=dev) / din ** 0.5
    dpre = torch.randn(B, dout, device=dev)
    outs8 = torch.empty(8, B, dout, device=dev)
    for tag, f in libs.items():
        res = {"tile": tag, "shape": f"{din}x{dout}", "smem_bytes": SMEM.get(tag)}
        for s in (4, 8, 16):
            ks = din // s
            out = torch.empty(s, B, dout, device=dev)
            fn = lambda s=s, ks=ks, out=out: f(0, 0, x.data_ptr(), din, ks, w.data_ptr(), dout, ks * dout,  # noqa
                                               out.data_ptr(), B, dout, ks, s, None, 0, cs())
            assert fn() == 0
            res[f"fwd_S{s}"] = t_graph(fn)
        gw = torch.empty(din, dout, device=dev)
        fn = lambda: f(1, 0, x.data_ptr(), din, 0, dpre.data_ptr(), dout, 0, gw.data_ptr(), din, dout, B, 1,  # noqa
                       None, 0, cs())
        assert fn() == 0
        res["wgrad"] = t_graph(fn)
        err = float((gw.double() - x.double().t() @ dpre.double()).abs().max() / gw.double().abs().max())
        res["wgrad_relerr"] = err
        for s in (2, 4, 8):
            ks = dout // s
            gi = torch.empty(s, B, din, device=dev)
            fn = lambda s=s, ks=ks, gi=gi: f(0, 1, dpre.data_ptr(), dout, ks, w.data_ptr(), dout, ks,  # noqa
                                             gi.data_ptr(), B, din, ks, s, None, 0, cs())
            assert fn() == 0
            res[f"dgrad_S{s}"] = t_graph(fn)
        res["conc4_fwd_S8_us_per_gemm"] = t_conc(lambda: f(0, 0, x.data_ptr(), din, din // 8, w.data_ptr(), dout,
                                                           din // 8 * dout, outs8.data_ptr(), B, dout, din // 8, 8,
                                                           None, 0, cs()))
        res["conc4_wgrad_us_per_gemm"] = t_conc(lambda: f(1, 0, x.data_ptr(), din, 0, dpre.data_ptr(), dout, 0,
                                                          gw.data_ptr(), din, dout, B, 1, None, 0, cs()))
        print(json.dumps(res), flush=True)
