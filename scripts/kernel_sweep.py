"""Kernel sweep: K1/K2/K3 x {sgdm, adam, adamw} x N, achieved algorithmic GB/s
against the measured HBM copy peak (MEASURED_PEAKS.json), CUDA-event timed
per launch with an L2 flush (256 MB read) between launches.

  python scripts/kernel_sweep.py                 # default sweep
  python scripts/kernel_sweep.py --tune          # launch-shape search at 2^28
  python scripts/kernel_sweep.py --sizes 30 --kinds adam --kernels step_predict
"""

from __future__ import annotations

import argparse
import ctypes
import itertools
import json
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2312_00839_b200 import _lib  # noqa: E402
from paper_2312_00839_b200.optim import OptimizerConfig  # noqa: E402

BYTES = {  # SURVEY.md §8d algorithmic bytes per fp32 parameter
    ("predict", "sgdm"): 12, ("predict", "adam"): 16, ("predict", "adamw"): 16,
    ("step", "sgdm"): 20, ("step", "adam"): 28, ("step", "adamw"): 28,
    ("step_predict", "sgdm"): 24, ("step_predict", "adam"): 32, ("step_predict", "adamw"): 32,
}


def peak_gbs() -> float:
    p = Path(__file__).resolve().parent.parent / "MEASURED_PEAKS.json"
    try:
        return float(json.loads(p.read_text())["hbm_gbs"])
    except Exception:
        return 6650.0  # B200_PROFILING.md fallback


class Buffers:
    def __init__(self, n: int, seed: int = 0):
        g = torch.Generator(device="cuda")
        dev = "cuda"
        self.n = n
        g.manual_seed(seed)
        self.w = torch.randn(n, device=dev, generator=g) * 0.02
        g.manual_seed(seed + 1)
        self.g = torch.randn(n, device=dev, generator=g) * 1e-2
        g.manual_seed(seed + 2)
        self.m = torch.randn(n, device=dev, generator=g) * 1e-3
        g.manual_seed(seed + 3)
        self.v = (torch.randn(n, device=dev, generator=g) * 1e-2).square_()
        self.out = torch.empty(n, device=dev)


def call(lib, kernel, kind, b: Buffers, launch, stream, t=10, s=3, lr=1e-3):
    hp = ctypes.byref(OptimizerConfig(kind).hparams())
    la = ctypes.byref(launch) if launch is not None else None
    v = None if kind == "sgdm" else b.v.data_ptr()
    if kernel == "predict":
        rc = lib.po_predict(hp, b.w.data_ptr(), b.m.data_ptr(), v, b.out.data_ptr(), b.n, lr * s, t,
                            la, stream)
    elif kernel == "step":
        rc = lib.po_step(hp, b.w.data_ptr(), b.g.data_ptr(), b.m.data_ptr(), v, None, b.n, lr, t,
                         None, la, stream)
    else:
        rc = lib.po_step_predict(hp, b.w.data_ptr(), b.g.data_ptr(), b.m.data_ptr(), v,
                                 b.out.data_ptr(), b.n, lr, lr * s, t, None, la, stream)
    _lib.check(rc, kernel)


FLUSH = True


def time_kernel(lib, kernel, kind, b, launch=None, reps=20, warmup=5):
    stream = torch.cuda.current_stream()
    # L2 flush by READING 256 MB (2x L2): clean lines, so the timed kernel does
    # not pay for write-backs of the flush itself
    flush = torch.ones(256 * 1024 * 1024 // 4, device="cuda")
    for _ in range(warmup):
        call(lib, kernel, kind, b, launch, stream.cuda_stream)
    times = []
    for _ in range(reps):
        if FLUSH:
            flush.sum()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        call(lib, kernel, kind, b, launch, stream.cuda_stream)
        e1.record(stream)
        e1.synchronize()
        times.append(e0.elapsed_time(e1) / 1e3)
    return statistics.median(times), min(times)


def copy_gbs(n: int) -> float:
    a = torch.empty(n, device="cuda")
    c = torch.empty(n, device="cuda")
    for _ in range(3):
        c.copy_(a)
    ts = []
    for _ in range(10):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        c.copy_(a)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) / 1e3)
    return 2 * 4 * n / min(ts) / 1e9


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="20,22,24,26,28,30", help="log2 sizes (or 'e9' for 1e9)")
    ap.add_argument("--kinds", default="sgdm,adam,adamw")
    ap.add_argument("--kernels", default="predict,step,step_predict")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--tune", action="store_true")
    ap.add_argument("--tune-log2", type=int, default=28)
    ap.add_argument("--tune-all", action="store_true",
                    help="focused launch-shape search for every kernel x kind")
    ap.add_argument("--out", default=None)
    ap.add_argument("--no-flush", action="store_true", help="warm L2 (pipeline-like) instead of flushing")
    ap.add_argument("--tune-small", action="store_true", help="launch-shape search at 2^20..2^24")
    ap.add_argument("--s-sweep", action="store_true",
                    help="K1/K3 x kinds at s = 1..7 (BASELINE configs[4]) at the first --sizes entry")
    args = ap.parse_args()
    global FLUSH
    FLUSH = not args.no_flush
    lib = _lib.load()
    peak = peak_gbs()
    rows = []
    print(f"# device {torch.cuda.get_device_name()}  measured copy peak {peak} GB/s", flush=True)
    if args.s_sweep:
        sz = args.sizes.split(",")[0]
        n = int(1e9) if sz == "e9" else 1 << int(sz)
        b = Buffers(n)
        for kind in args.kinds.split(","):
            for kernel in ("predict", "step_predict"):
                for s_ in range(1, 8):
                    stream = torch.cuda.current_stream()
                    call(lib, kernel, kind, b, None, stream.cuda_stream, s=s_)
                    times = []
                    for _ in range(args.reps):
                        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        e0.record(stream)
                        call(lib, kernel, kind, b, None, stream.cuda_stream, s=s_)
                        e1.record(stream)
                        e1.synchronize()
                        times.append(e0.elapsed_time(e1) / 1e3)
                    med = statistics.median(times)
                    gbs = BYTES[(kernel, kind)] * n / med / 1e9
                    row = dict(n=n, kind=kind, kernel=kernel, s=s_, ms_median=round(med * 1e3, 4), gbs=round(gbs, 1),
                               frac_of_measured=round(gbs / peak, 4))
                    rows.append(row)
                    print(json.dumps(row), flush=True)
    elif args.tune_small:
        shapes = [(512, 1, 1), (512, 2, 1), (512, 4, 1), (256, 8, 1), (256, 4, 2), (128, 16, 1), (512, 2, 2),
                  (256, 8, 2), (128, 16, 2), (256, 6, 1), (128, 8, 1), (128, 8, 2), (128, 8, 4), (256, 4, 4),
                  (512, 2, 4), (512, 1, 4), (256, 2, 4)]
        for lg in (20, 22, 24):
            n = 1 << lg
            b = Buffers(n)
            for kernel in args.kernels.split(","):
                for kind in args.kinds.split(","):
                    for (block, cps, unroll), cache in itertools.product([(None, None, None)] + shapes, (1, 4)):
                        if block is None and cache == 4:
                            continue
                        la = None if block is None else _lib.make_launch(block, cps, 8, cache, unroll)
                        med, best = time_kernel(lib, kernel, kind, b, la, reps=20, warmup=3)
                        gbs = BYTES[(kernel, kind)] * n / med / 1e9
                        row = dict(n=n, kernel=kernel, kind=kind, block=block, cps=cps, unroll=unroll, cache=cache,
                                   us=round(med * 1e6, 2), gbs=round(gbs, 1), frac=round(gbs / peak, 4),
                                   flush=FLUSH)
                        rows.append(row)
                        print(json.dumps(row), flush=True)
    elif args.tune_all:
        n = 1 << args.tune_log2
        b = Buffers(n)
        print(f"# torch copy_ at 2^{args.tune_log2}: {copy_gbs(n):.1f} GB/s", flush=True)
        shapes = [(512, 1, 1), (512, 2, 1), (256, 2, 1), (256, 4, 1), (384, 1, 1), (1024 // 2, 1, 2),
                  (128, 16, 2), (128, 8, 2), (256, 8, 2), (256, 4, 2), (128, 12, 2), (192, 8, 2),
                  (128, 16, 1), (256, 6, 1), (128, 24, 1)]
        for kernel in args.kernels.split(","):
            for kind in args.kinds.split(","):
                for block, cps, unroll in shapes:
                    for cache in (1, 3):
                        la = _lib.make_launch(block, cps, 8, cache, unroll)
                        med, best = time_kernel(lib, kernel, kind, b, la, reps=10, warmup=2)
                        gbs = BYTES[(kernel, kind)] * n / med / 1e9
                        row = dict(kernel=kernel, kind=kind, unroll=unroll, cache=cache, block=block,
                                   cps=cps, ms=med * 1e3, gbs=round(gbs, 1), frac=round(gbs / peak, 4))
                        rows.append(row)
                        print(json.dumps(row), flush=True)
    elif args.tune:
        n = 1 << args.tune_log2
        b = Buffers(n)
        print(f"# torch copy_ at 2^{args.tune_log2}: {copy_gbs(n):.1f} GB/s", flush=True)
        for kind in ("adam", "sgdm"):
            for vec in (8, 4):
                for unroll in (1, 2, 4):
                    for cache in (1, 2, 3):
                        for block, cps in ((256, 4), (256, 8), (512, 2), (512, 1), (128, 8), (128, 16), (512, 4)):
                            la = _lib.make_launch(block, cps, vec, cache, unroll)
                            med, best = time_kernel(lib, "step_predict", kind, b, la, reps=8, warmup=2)
                            gbs = BYTES[("step_predict", kind)] * n / med / 1e9
                            row = dict(kind=kind, vec=vec, unroll=unroll, cache=cache, block=block,
                                       cps=cps, ms=med * 1e3, gbs=round(gbs, 1), frac=round(gbs / peak, 4))
                            rows.append(row)
                            print(json.dumps(row), flush=True)
    else:
        for sz in args.sizes.split(","):
            n = int(1e9) if sz == "e9" else 1 << int(sz)
            b = Buffers(n)
            for kind in args.kinds.split(","):
                for kernel in args.kernels.split(","):
                    med, best = time_kernel(lib, kernel, kind, b, reps=args.reps)
                    gbs = BYTES[(kernel, kind)] * n / med / 1e9
                    row = dict(n=n, kind=kind, kernel=kernel, ms_median=round(med * 1e3, 4),
                               ms_best=round(best * 1e3, 4), gbs=round(gbs, 1),
                               frac_of_measured=round(gbs / peak, 4), frac_of_8tbs=round(gbs / 8000, 4))
                    rows.append(row)
                    print(json.dumps(row), flush=True)
            del b
            torch.cuda.empty_cache()
    if args.out:
        Path(args.out).write_text("\n".join(json.dumps(r) for r in rows) + "\n")


if __name__ == "__main__":
    main()
