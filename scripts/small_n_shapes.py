"""K2/K3 (Adam) launch shapes at pipeline-stage sizes, timed as CUDA-graph
replays of back-to-back launches (no host overhead; the stage's buffers stay
warm in L2 as they do between a pipeline stage's updates)."""
import itertools
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2312_00839_b200 import _lib  # noqa: E402
from paper_2312_00839_b200.optim import FlatParams, OptimizerConfig, OptimizerState  # noqa: E402

dev = torch.device("cuda", 0)
for n in [int(v) for v in (sys.argv[1:] or ["3146752", "1049600"])]:
    flat = FlatParams.from_tensors(["w"], [torch.randn(n) * 0.02], dev)
    flat.grad.normal_(0, 1e-2)
    staging = flat.layout.empty(dev)
    best = {}
    for mode in ("k2", "k3"):
        rows = []
        shapes = [(None,)] + list(itertools.product((128, 256, 512), (1, 2, 4, 8, 16), (1, 2), (1, 3)))
        for sh in shapes:
            if sh != (None,) and sh[0] * sh[1] > 2048:
                continue
            la = None if sh == (None,) else _lib.make_launch(sh[0], sh[1], 8, sh[3], sh[2])
            opt = OptimizerState(OptimizerConfig("adam"), ["w"], device=dev, launch=la, eager_checks=False)
            fn = (lambda o=opt: o.step_predict_(flat, 1e-4, 1e-4, 3, staging)) if mode == "k3" else \
                (lambda o=opt: o.step_(flat, 1e-4))
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                for _ in range(20):
                    fn()
            g.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(5):
                g.replay()
            e1.record()
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) * 1e3 / 100
            rows.append((us, sh))
            g.keepalive = opt
            del g
        rows.sort()
        default = [r for r in rows if r[1] == (None,)][0]
        print(json.dumps({"n": n, "mode": mode, "default_us": round(default[0], 2),
                          "best": [(round(u, 2), s) for u, s in rows[:6]]}), flush=True)
