"""Three-piece pre-split (a = p0 + p1 + p2, bf16 each, ~24 mantissa bits)
with the six products that carry fp32-level accuracy (p0q0, p0q1, p1q0,
p0q2, p1q1, p2q0) as ONE cuBLASLt bf16 GEMM with fp32 output over a
K-concatenated operand pair (K' = 6K), vs po_gemm_f32x3, at the config-1
stage shapes. Accuracy vs float64; CUDA-graph timing (16 calls per graph)."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2312_00839_b200 import _lib  # noqa: E402
from presplit_gemm_probe import t_graph, relerr, emit  # noqa: E402

torch.backends.cuda.matmul.allow_tf32 = False
dev = torch.device("cuda", 0)
lib = _lib.load()
cs = lambda: torch.cuda.current_stream().cuda_stream  # noqa: E731
A_IDX, B_IDX = (0, 0, 1, 0, 1, 2), (0, 1, 0, 2, 1, 0)


def split3(a):
    p0 = a.to(torch.bfloat16)
    r = a - p0.float()
    p1 = r.to(torch.bfloat16)
    p2 = (r - p1.float()).to(torch.bfloat16)
    return p0, p1, p2


B = 128
for din, dout in ((3072, 1024), (1024, 1024)):
    x = torch.randn(B, din, device=dev)
    w = torch.randn(din, dout, device=dev) / din ** 0.5
    dpre = torch.randn(B, dout, device=dev)
    ref_f = x.double() @ w.double()
    ref_w = x.double().t() @ dpre.double()
    xp, wp, dp = split3(x), split3(w), split3(dpre)
    # forward: (B, 6K) . (6K, N)
    a_cat = torch.cat([xp[i] for i in A_IDX], 1).contiguous()
    b_cat = torch.cat([wp[i] for i in B_IDX], 0).contiguous()
    o1 = torch.empty(B, dout, device=dev)

    def kcat():
        torch.mm(a_cat, b_cat, out_dtype=torch.float32, out=o1)

    kcat()
    emit(case=f"fwd {din}x{dout}", form="bf16 6-product kcat mm", us=t_graph(kcat), relerr=relerr(o1, ref_f))
    for s in (1, 2, 4):
        ks = din // s
        a6 = torch.stack([xp[i] for i in A_IDX]).view(6, B, s, ks).permute(0, 2, 1, 3).reshape(6 * s, B, ks).contiguous()
        b6 = torch.stack([wp[i] for i in B_IDX]).view(6 * s, ks, dout).contiguous()
        o6 = torch.empty(6 * s, B, dout, device=dev)

        def bat(a6=a6, b6=b6, o6=o6):
            torch.bmm(a6, b6, out_dtype=torch.float32, out=o6)

        bat()
        emit(case=f"fwd {din}x{dout}", form=f"bf16 6-product bmm 6xS{s}", us=t_graph(bat),
             relerr=relerr(o6.double().sum(0), ref_f))
    # weight gradient: (K_in, 6B) . (6B, N), A read transposed from the (6B, K_in) stash
    xcat = torch.cat([xp[i] for i in A_IDX], 0).contiguous()
    dcat = torch.cat([dp[i] for i in B_IDX], 0).contiguous()
    gw = torch.empty(din, dout, device=dev)

    def wg():
        torch.mm(xcat.t(), dcat, out_dtype=torch.float32, out=gw)

    wg()
    emit(case=f"wgrad {din}x{dout}", form="bf16 6-product kcat mm", us=t_graph(wg), relerr=relerr(gw, ref_w))
    gw32 = torch.empty(din, dout, device=dev)

    def wg32():
        assert lib.po_gemm_f32x3(1, 0, x.data_ptr(), din, 0, dpre.data_ptr(), dout, 0, gw32.data_ptr(), din, dout, B,
                                 1, None, 0, cs()) == 0

    wg32()
    emit(case=f"wgrad {din}x{dout}", form="f32x3", us=t_graph(wg32), relerr=relerr(gw32, ref_w))
    # input gradient: dpre (B, 6N) . W^T pieces (6N, K_in) read transposed from (K_in, 6N)?  W pieces are
    # (K_in, N) each; concat along N -> (K_in, 6N), transposed view -> (6N, K_in)
    dcat_k = torch.cat([dp[i] for i in A_IDX], 1).contiguous()
    wcat_n = torch.cat([wp[i] for i in B_IDX], 1).contiguous()
    gi = torch.empty(B, din, device=dev)

    def dg():
        torch.mm(dcat_k, wcat_n.t(), out_dtype=torch.float32, out=gi)

    dg()
    emit(case=f"dgrad {din}x{dout}", form="bf16 6-product kcat mm", us=t_graph(dg),
         relerr=relerr(gi, dpre.double() @ w.double().t()))
