"""Pre-split bf16 operands + cuBLASLt bf16 GEMM (fp32 out) vs po_gemm_f32x3
(CUTLASS fast-FP32, split in shared memory) on the config-1 stage shapes.

Each fp32 operand a = hi + lo (hi = bf16(a), lo = bf16(a - hi)); the three
products hi.hi + hi.lo + lo.hi are one bf16 GEMM over a K-concatenated
operand pair [a_hi | a_hi | a_lo] . [b_hi ; b_lo ; b_hi] (K' = 3K), or a
batched GEMM with the split-K slices x 3 products as the batch. The split
itself is timed separately (torch elementwise here; a fused kernel would do
it in the producer's epilogue). Accuracy vs float64 and CUDA-graph timing
(16 back-to-back calls per graph)."""
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


def t_graph(fn, reps=16):
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
    best = 1e9
    for _ in range(5):
        e0.record()
        for _ in range(10):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e3 / (10 * reps))
    return round(best, 2)


def split(a):
    hi = a.to(torch.bfloat16)
    lo = (a - hi.float()).to(torch.bfloat16)
    return hi, lo


def relerr(got, ref):
    return float((got.double() - ref).abs().max() / ref.abs().max())


def emit(**kw):
    print(json.dumps(kw), flush=True)



def main():
    B = 128
    for din, dout in ((3072, 1024), (1024, 1024)):
        x = torch.randn(B, din, device=dev)
        w = torch.randn(din, dout, device=dev) / din ** 0.5
        dpre = torch.randn(B, dout, device=dev)
        ref_f = x.double() @ w.double()
        ref_w = x.double().t() @ dpre.double()
        xh, xl = split(x)
        wh, wl = split(w)
        dh, dl = split(dpre)

        # --- forward: current path (split-K 8 fast-FP32 + partial sum)
        s = 8
        ks = din // s
        out = torch.empty(s, B, dout, device=dev)

        def f32x3(s=s, ks=ks, out=out):
            assert lib.po_gemm_f32x3(0, 0, x.data_ptr(), din, ks, w.data_ptr(), dout, ks * dout, out.data_ptr(), B,
                                     dout, ks, s, None, 0, cs()) == 0

        f32x3()
        emit(case=f"fwd {din}x{dout}", form="f32x3 S8", us=t_graph(f32x3), relerr=relerr(out.sum(0), ref_f))

        # --- forward: K-concatenated single bf16 GEMM, fp32 out
        a_cat = torch.cat([xh, xh, xl], 1).contiguous()          # (B, 3K)
        b_cat = torch.cat([wh, wl, wh], 0).contiguous()          # (3K, N)
        o1 = torch.empty(B, dout, device=dev)

        def kcat():
            torch.mm(a_cat, b_cat, out_dtype=torch.float32, out=o1)

        try:
            kcat()
            emit(case=f"fwd {din}x{dout}", form="bf16 kcat mm", us=t_graph(kcat), relerr=relerr(o1, ref_f))
        except Exception as exc:  # noqa: BLE001
            emit(case=f"fwd {din}x{dout}", form="bf16 kcat mm", error=str(exc)[:200])

        # --- forward: batched split-K slices x 3 products
        for s in (1, 2, 4, 8):
            ks = din // s
            a3 = torch.stack([xh, xh, xl]).view(3, B, s, ks).permute(0, 2, 1, 3).reshape(3 * s, B, ks).contiguous()
            b3 = torch.stack([wh, wl, wh]).view(3, s, ks, dout).reshape(3 * s, ks, dout).contiguous()
            o3 = torch.empty(3 * s, B, dout, device=dev)

            def bat(a3=a3, b3=b3, o3=o3):
                torch.bmm(a3, b3, out_dtype=torch.float32, out=o3)

            try:
                bat()
                emit(case=f"fwd {din}x{dout}", form=f"bf16 bmm 3xS{s}", us=t_graph(bat), relerr=relerr(o3.sum(0), ref_f))
            except Exception as exc:  # noqa: BLE001
                emit(case=f"fwd {din}x{dout}", form=f"bf16 bmm 3xS{s}", error=str(exc)[:200])

        # --- weight gradient: current path
        gw = torch.empty(din, dout, device=dev)

        def wg32():
            assert lib.po_gemm_f32x3(1, 0, x.data_ptr(), din, 0, dpre.data_ptr(), dout, 0, gw.data_ptr(), din, dout, B, 1,
                                     None, 0, cs()) == 0

        wg32()
        emit(case=f"wgrad {din}x{dout}", form="f32x3", us=t_graph(wg32), relerr=relerr(gw, ref_w))
        xcat_t = torch.cat([xh, xh, xl], 0)                      # (3B, K) -> transposed view (K, 3B)
        dcat = torch.cat([dh, dl, dh], 0)                        # (3B, N)
        gw2 = torch.empty(din, dout, device=dev)

        def wgcat():
            torch.mm(xcat_t.t(), dcat, out_dtype=torch.float32, out=gw2)

        try:
            wgcat()
            emit(case=f"wgrad {din}x{dout}", form="bf16 kcat mm", us=t_graph(wgcat), relerr=relerr(gw2, ref_w))
        except Exception as exc:  # noqa: BLE001
            emit(case=f"wgrad {din}x{dout}", form="bf16 kcat mm", error=str(exc)[:200])

        # --- the split itself (torch elementwise; upper bound for a fused kernel)
        def sp_act():
            split(x)

        def sp_w():
            split(w)

        emit(case=f"split {din}x{dout}", form="torch act", us=t_graph(sp_act))
        emit(case=f"split {din}x{dout}", form="torch weight", us=t_graph(sp_w))


if __name__ == "__main__":
    main()
