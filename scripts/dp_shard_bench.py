"""One-GPU timing of the three K3 forms at dp = 1 (all replicas local):
plain K3 (po_step_predict), the peer-load DP kernel (po_step_predict_dp) and
the sharded DP kernel (po_step_predict_dp_shard, with its wait / done
kernels), CUDA events, inputs >> L2. At dp = 1 every form moves the same 32
B/param, so this isolates each kernel's HBM efficiency; the dp > 1 costs are
NVLink-bound and are modelled in DESIGN.md §3.

  python scripts/dp_shard_bench.py [--n 1e9] [--kind adam]
"""
import argparse
import ctypes
import json
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2312_00839_b200 import _lib  # noqa: E402
from paper_2312_00839_b200.optim import OptimizerConfig  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=float, default=1e9)
ap.add_argument("--kind", default="adam")
ap.add_argument("--reps", type=int, default=10)
a = ap.parse_args()
n = int(a.n)
dev = torch.device("cuda", 0)
lib = _lib.load()
hp = ctypes.byref(OptimizerConfig(a.kind).hparams())
g = torch.Generator(device=dev).manual_seed(0)
w = torch.randn(n, device=dev, generator=g) * 0.02
gr = torch.randn(n, device=dev, generator=g) * 1e-2
m = torch.randn(n, device=dev, generator=g) * 1e-3
v = (torch.randn(n, device=dev, generator=g) * 1e-2).square_()
out = torch.empty(n, device=dev)
bad = torch.full((1,), 2 ** 63 - 1, dtype=torch.int64, device=dev)
flags = torch.full((1,), 2 ** 62, dtype=torch.int64, device=dev)  # every epoch already signalled
done = torch.zeros(1, dtype=torch.int64, device=dev)
done_slots = torch.tensor([done.data_ptr()], dtype=torch.int64, device=dev)
status = torch.zeros(1, dtype=torch.int32, device=dev)
P1 = ctypes.c_void_p * 1
stream = torch.cuda.current_stream().cuda_stream
s2 = None if a.kind == "sgdm" else v.data_ptr()
epoch = [0]


def k3():
    return lib.po_step_predict(hp, w.data_ptr(), gr.data_ptr(), m.data_ptr(), s2, out.data_ptr(), n, 1e-4, 3e-4, 5,
                               bad.data_ptr(), None, stream)


def dp_load():
    return lib.po_step_predict_dp(hp, w.data_ptr(), P1(gr.data_ptr()), 1, m.data_ptr(), s2, out.data_ptr(), n, 1e-4,
                                  3e-4, 5, bad.data_ptr(), flags.data_ptr(), 1, 10_000, status.data_ptr(), stream)


def dp_shard():
    epoch[0] += 1
    return lib.po_step_predict_dp_shard(hp, 1, 0, P1(w.data_ptr()), P1(gr.data_ptr()), P1(m.data_ptr()),
                                        None if s2 is None else P1(s2), P1(out.data_ptr()), n, 1e-4, 3e-4, 5, None,
                                        P1(bad.data_ptr()), flags.data_ptr(), done_slots.data_ptr(), done.data_ptr(),
                                        epoch[0], None, 10_000, status.data_ptr(), None, stream)


bytes_per = 24 if a.kind == "sgdm" else 32
res = {}
for _ in range(3):  # alternate the forms trial by trial
    for name, fn in (("k3", k3), ("dp_peer_load", dp_load), ("dp_shard", dp_shard)):
        for _ in range(2):
            _lib.check(fn(), name)
        ts = []
        for _ in range(a.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            _lib.check(fn(), name)
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1) / 1e3)
        res.setdefault(name, []).append(statistics.median(ts))
assert int(status.item()) == 0
for name, tl in res.items():
    t = statistics.median(tl)
    print(json.dumps({"form": name, "kind": a.kind, "n": n, "dp": 1, "ms": round(t * 1e3, 4),
                      "gbs": round(bytes_per * n / t / 1e9, 1)}), flush=True)
