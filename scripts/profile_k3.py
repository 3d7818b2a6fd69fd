"""Minimal driver for an ncu capture of the predictor/optimizer kernels:
allocates one stage's flat buffers and launches the chosen kernel a few times.

  ncu --set full --clock-control none --import-source on -k regex:po_stream_kernel \
      -s 2 -c 1 -o gpurun_out/k3 python scripts/profile_k3.py --n 268435456 --kind adam
"""

import argparse
import ctypes
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2312_00839_b200 import _lib  # noqa: E402
from paper_2312_00839_b200.optim import OptimizerConfig  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1 << 28)
    ap.add_argument("--kind", default="adam")
    ap.add_argument("--kernel", default="step_predict", choices=["step_predict", "step", "predict"])
    ap.add_argument("--launches", type=int, default=4)
    a = ap.parse_args()
    lib = _lib.load()
    n = a.n
    g = torch.Generator(device="cuda").manual_seed(0)
    w = torch.randn(n, device="cuda", generator=g) * 0.02
    gr = torch.randn(n, device="cuda", generator=g) * 1e-2
    m = torch.randn(n, device="cuda", generator=g) * 1e-3
    v = (torch.randn(n, device="cuda", generator=g) * 1e-2).square_()
    out = torch.empty(n, device="cuda")
    hp = ctypes.byref(OptimizerConfig(a.kind).hparams())
    vp = None if a.kind == "sgdm" else v.data_ptr()
    st = torch.cuda.current_stream().cuda_stream
    for i in range(a.launches):
        if a.kernel == "step_predict":
            rc = lib.po_step_predict(hp, w.data_ptr(), gr.data_ptr(), m.data_ptr(), vp, out.data_ptr(), n, 1e-3,
                                     3e-3, 10 + i, None, None, st)
        elif a.kernel == "step":
            rc = lib.po_step(hp, w.data_ptr(), gr.data_ptr(), m.data_ptr(), vp, None, n, 1e-3, 10 + i, None,
                             None, st)
        else:
            rc = lib.po_predict(hp, w.data_ptr(), m.data_ptr(), vp, out.data_ptr(), n, 3e-3, 10 + i, None, st)
        _lib.check(rc, a.kernel)
    torch.cuda.synchronize()
    print("done", a.kernel, a.kind, n)


if __name__ == "__main__":
    main()
