"""A/B of the optimizer-kernel arithmetic and loop structure on ONE box.

Builds (here, `--build`) two standalone copies of pipeoptim_kernels.cu into
paper_2312_00839_b200/build/probe/: `new` (the shipped source) and `div3`
(-DPO_PROBE_ADAM_DIV3: the round-1 three-division Adam direction, timing
only — its results are not the shipped rounding). On the GPU box it times
K1/K2/K3 for the listed kinds at the listed sizes for each library x launch
shape, alternating libraries trial by trial so clock/thermal drift cancels,
and prints one JSON line per (lib, kernel, kind, n, shape).

  python scripts/adam_dir_ab.py --build                       # here
  python scripts/adam_dir_ab.py --sizes e9 --out gpurun_out/ab.jsonl   # box
"""

from __future__ import annotations

import argparse
import ctypes
import json
import statistics
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
PROBE = ROOT / "paper_2312_00839_b200" / "build" / "probe"
VARIANTS = {"new": [], "div3": ["-DPO_PROBE_ADAM_DIV3"]}


def build():
    from paper_2312_00839_b200.build import ARCH_FLAGS, NVCC_FLAGS, nvcc_path

    PROBE.mkdir(parents=True, exist_ok=True)
    src = ROOT / "paper_2312_00839_b200" / "csrc" / "pipeoptim_kernels.cu"
    procs = []
    for name, flags in VARIANTS.items():
        cmd = [nvcc_path(), *ARCH_FLAGS, *NVCC_FLAGS, f"-I{ROOT / 'include'}", *flags, "-shared", "-o",
               str(PROBE / f"libk_{name}.so"), str(src), "-lcuda"]
        procs.append(subprocess.Popen(cmd))
    assert all(p.wait() == 0 for p in procs)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--build", action="store_true")
    ap.add_argument("--sizes", default="e9")
    ap.add_argument("--kinds", default="adam,sgdm")
    ap.add_argument("--kernels", default="step_predict,step,predict")
    ap.add_argument("--shapes", default="0:0:0,512:1:1,512:1:3,256:2:3,256:2:1,384:1:3,512:1:2,128:16:1,128:16:3",
                    help="block:ctas_per_sm:unroll, 0:0:0 = the library default")
    ap.add_argument("--libs", default="new,div3")
    ap.add_argument("--trials", type=int, default=5)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--flush", action="store_true", help="L2 flush (256 MB read) before every launch")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    if args.build:
        build()
        return
    import torch

    sys.path.insert(0, str(ROOT / "scripts"))
    import kernel_sweep as ks
    from paper_2312_00839_b200 import _lib
    from paper_2312_00839_b200.optim import OptimizerConfig  # noqa: F401

    libs = {}
    for name in args.libs.split(","):
        lib = ctypes.CDLL(str(PROBE / f"libk_{name}.so"))
        for fn in ("po_step", "po_predict", "po_step_predict"):
            getattr(lib, fn).restype, getattr(lib, fn).argtypes = _lib._SIGNATURES[fn]
        libs[name] = lib
    peak = ks.peak_gbs()
    out = open(args.out, "a") if args.out else None
    flush = torch.ones(256 * 1024 * 1024 // 4, device="cuda") if args.flush else None
    stream = torch.cuda.current_stream()
    sizes = [1_000_000_000 if s == "e9" else 1 << int(s) for s in args.sizes.split(",")]
    shapes = [tuple(int(x) for x in s.split(":")) for s in args.shapes.split(",")]
    for n in sizes:
        b = ks.Buffers(n)
        for kind in args.kinds.split(","):
            for kernel in args.kernels.split(","):
                times = {(ln, sh): [] for ln in libs for sh in shapes}
                for _ in range(args.trials):
                    for sh in shapes:
                        la = None if sh == (0, 0, 0) else _lib.make_launch(block=sh[0], ctas_per_sm=sh[1],
                                                                           unroll=sh[2])
                        for ln, lib in libs.items():
                            for _ in range(2):
                                ks.call(lib, kernel, kind, b, la, stream.cuda_stream)
                            ts = []
                            for _ in range(args.reps):
                                if flush is not None:
                                    flush.sum()
                                e0 = torch.cuda.Event(enable_timing=True)
                                e1 = torch.cuda.Event(enable_timing=True)
                                e0.record(stream)
                                ks.call(lib, kernel, kind, b, la, stream.cuda_stream)
                                e1.record(stream)
                                e1.synchronize()
                                ts.append(e0.elapsed_time(e1) / 1e3)
                            times[(ln, sh)].append(statistics.median(ts))
                for (ln, sh), tl in times.items():
                    t = statistics.median(tl)
                    gbs = ks.BYTES[(kernel, kind)] * n / t / 1e9
                    rec = {"n": n, "kernel": kernel, "kind": kind, "lib": ln, "shape": list(sh),
                           "us": round(t * 1e6, 2), "gbs": round(gbs, 1), "frac": round(gbs / peak, 4),
                           "flush": bool(args.flush)}
                    print(json.dumps(rec), flush=True)
                    if out:
                        out.write(json.dumps(rec) + "\n")
        del b
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
