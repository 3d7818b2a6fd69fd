"""Forward GEMM of the config-1 layers (M = B = 128 rows, long K, few output
tiles): cuBLAS mm vs split-K bmm + reduction vs the transposed problem."""
import json

import torch

from gemm_variants import t_graph  # noqa: F401  (same timing helper)

torch.backends.cuda.matmul.allow_tf32 = False
dev = torch.device("cuda", 0)
B = 128
for din, dout in ((3072, 1024), (1024, 1024), (1024, 10)):
    x = torch.randn(B, din, device=dev)
    w = torch.randn(din, dout, device=dev) * 0.02
    wt = w.t().contiguous()
    res = {"mm": t_graph(lambda: torch.mm(x, w)), "transposed": t_graph(lambda: torch.mm(wt, x.t()))}
    for S in (2, 4, 8, 16, 32):
        if din % S:
            continue
        xs = x.view(B, S, din // S).transpose(0, 1)  # (S, B, K/S) strided view
        ws = w.view(S, din // S, dout)
        res[f"splitk{S}"] = t_graph(lambda xs=xs, ws=ws: torch.bmm(xs, ws).sum(0))
        res[f"splitk{S}_bmm_only"] = t_graph(lambda xs=xs, ws=ws: torch.bmm(xs, ws))
    ref = torch.mm(x.double(), w.double())
    err = {f"splitk{S}": float((torch.bmm(x.view(B, S, din // S).transpose(0, 1), w.view(S, din // S, dout)).sum(0)
                                .double() - ref).abs().max()) for S in (4, 8) if din % S == 0}
    err["mm"] = float((torch.mm(x, w).double() - ref).abs().max())
    print(json.dumps({"shape": [B, din, dout], "us": {k: round(v, 2) for k, v in res.items()}, "maxerr": err}),
          flush=True)
