"""K1/K2/K3 at pipeline-stage sizes, timed as CUDA-graph replays of
back-to-back launches that ROTATE over enough buffer sets that the working set
is > 2x L2 ("for N <= 2^24, rotate >= 8 buffer sets or flush
L2"): every launch streams cold data from HBM, and no per-launch host or
event overhead is included. `--warm` times one buffer set instead (the
L2-resident case of a pipeline stage updated again and again).

  python scripts/small_n_graph.py [--warm] [--sizes 20,22,24] [--out f.jsonl]
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
from paper_2312_00839_b200.roofline import peaks  # noqa: E402

BYTES = {"predict": (12, 16), "step": (20, 28), "step_predict": (24, 32)}
L2 = 126 * 2**20


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="20,22,24")
    ap.add_argument("--kinds", default="sgdm,adam,adamw")
    ap.add_argument("--kernels", default="predict,step,step_predict")
    ap.add_argument("--warm", action="store_true")
    ap.add_argument("--shape", default=None, help="block,ctas_per_sm,unroll,cache (default: tuned)")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    lib = _lib.load()
    peak = peaks()["hbm_gbs"]
    la = None
    if a.shape:
        b, c, u, ca = (int(x) for x in a.shape.split(","))
        la = ctypes.byref(_lib.make_launch(b, c, 8, ca, u))
    rows = []
    for lg in (int(x) for x in a.sizes.split(",")):
        n = 1 << lg
        per_set = 5 * 4 * n
        sets = 1 if a.warm else max(2, -(-3 * L2 // per_set))
        bufs = []
        for i in range(sets):
            g = torch.Generator(device="cuda").manual_seed(i)
            bufs.append(dict(w=torch.randn(n, device="cuda", generator=g) * 0.02,
                             g=torch.randn(n, device="cuda", generator=g) * 1e-2,
                             m=torch.randn(n, device="cuda", generator=g) * 1e-3,
                             v=(torch.randn(n, device="cuda", generator=g) * 1e-2).square_(),
                             o=torch.empty(n, device="cuda")))
        launches = max(16, 2 * sets)
        for kind in a.kinds.split(","):
            hp = ctypes.byref(OptimizerConfig(kind).hparams())
            for kernel in a.kernels.split(","):
                def one(b):
                    st = torch.cuda.current_stream()  # the capture stream inside torch.cuda.graph
                    v = None if kind == "sgdm" else b["v"].data_ptr()
                    if kernel == "predict":
                        rc = lib.po_predict(hp, b["w"].data_ptr(), b["m"].data_ptr(), v, b["o"].data_ptr(), n,
                                            3e-3, 10, la, st.cuda_stream)
                    elif kernel == "step":
                        rc = lib.po_step(hp, b["w"].data_ptr(), b["g"].data_ptr(), b["m"].data_ptr(), v, None, n,
                                         1e-3, 10, None, la, st.cuda_stream)
                    else:
                        rc = lib.po_step_predict(hp, b["w"].data_ptr(), b["g"].data_ptr(), b["m"].data_ptr(), v,
                                                 b["o"].data_ptr(), n, 1e-3, 3e-3, 10, None, la, st.cuda_stream)
                    _lib.check(rc, kernel)

                for i in range(sets):
                    one(bufs[i])
                torch.cuda.synchronize()
                graph = torch.cuda.CUDAGraph()
                with torch.cuda.graph(graph):
                    for i in range(launches):
                        one(bufs[i % sets])
                graph.replay()
                torch.cuda.synchronize()
                ts = []
                for _ in range(7):
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    graph.replay()
                    e1.record()
                    torch.cuda.synchronize()
                    ts.append(e0.elapsed_time(e1) / 1e3 / launches)
                ts.sort()
                sec = ts[len(ts) // 2]
                bpp = BYTES[kernel][0 if kind == "sgdm" else 1]
                gbs = bpp * n / sec / 1e9
                row = dict(n=n, kind=kind, kernel=kernel, us=round(sec * 1e6, 2), gbs=round(gbs, 1),
                           frac=round(gbs / peak, 4), sets=sets, l2=("warm (one set)" if a.warm else
                                                                    f"cold ({sets} rotating sets > 2x L2)"),
                           shape=a.shape or "default")
                rows.append(row)
                print(json.dumps(row), flush=True)
                del graph
        del bufs
        torch.cuda.empty_cache()
    if a.out:
        Path(a.out).write_text("".join(json.dumps(r) + "\n" for r in rows))


if __name__ == "__main__":
    main()
