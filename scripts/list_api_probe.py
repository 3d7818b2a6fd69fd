"""Where the reference-shaped list API's time goes (e2e.list_api): the three
calls of one step timed separately on pinned host tensors, plus the raw
pinned allocation cost."""
import json
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2312_00839_b200.optim import OptimizerConfig, OptimizerState, predict_weights  # noqa: E402

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 250_000_000
dev = torch.device("cuda", 0)
w = torch.empty(n).pin_memory().normal_(0, 0.02)
g = torch.empty(n).pin_memory().normal_(0, 1e-2)
opt = OptimizerState(OptimizerConfig("adam"), ["flat"], device=dev, eager_checks=False)


def t(fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = fn()
    torch.cuda.synchronize()
    return r, (time.perf_counter() - t0) * 1e3


for it in range(5):
    (new, dirs), a = t(lambda: opt.step([w], [g], 1e-3))
    d, b = t(lambda: opt.prediction_direction(new))
    wh, c = t(lambda: predict_weights(new, 1e-3, 3, d))
    del new, dirs, d, wh  # the bench's pattern: nothing outlives the step
    _, p = t(lambda: torch.empty(n, dtype=torch.float32, pin_memory=True))
    print(json.dumps({"iter": it, "n": n, "step_ms": round(a, 1), "direction_ms": round(b, 1),
                      "predict_weights_ms": round(c, 1), "pinned_alloc_ms": round(p, 1)}), flush=True)
