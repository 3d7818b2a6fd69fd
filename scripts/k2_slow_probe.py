"""Why is K2 slow inside the config-1 stage-0 unit graph (ncu: 175 us vs K3
16 us)? Replays the pred-off unit graph, then times K2 and K3 eagerly on
copies of the same W, G, m, v and reports their value ranges."""
import ctypes
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2312_00839_b200 import _lib  # noqa: E402
from paper_2312_00839_b200 import bench_pipeline as bp  # noqa: E402
from paper_2312_00839_b200.optim import OptimizerConfig, OptimizerState  # noqa: E402
from paper_2312_00839_b200.stages import build_layers, build_stages, torch_init  # noqa: E402

torch.backends.cuda.matmul.allow_tf32 = False
dev = torch.device("cuda", 0)
data = bp.DeviceBatches(torch, dev)
lib = _lib.load()
for key in ("pred_off", "pred_on"):
    st = build_stages(build_layers(bp.CONFIG1_DIMS, bp.CONFIG1_ACTS), 4, torch_init(7, dev), device=dev)
    opts = [OptimizerState(OptimizerConfig("adam"), s.param_names, device=dev) for s in st]
    g = bp._unit_graph(torch, dev, 0, st[0], opts[0], data, "softmax_xent", key == "pred_on", 4)
    for _ in range(40):
        g.replay()
    torch.cuda.synchronize()
    o, f = opts[0], st[0].flat

    def stats(t):
        a = t.abs()
        nz = a[a > 0]
        return {"min_nz": float(nz.min()) if nz.numel() else 0.0, "max": float(a.max()),
                "denormal": int(((a > 0) & (a < 1.1754944e-38)).sum()), "zero": int((a == 0).sum()),
                "nonfinite": int((~torch.isfinite(t)).sum())}

    rep = {"key": key, "step_count": o.step_count, "W": stats(f.data), "G": stats(f.grad), "m": stats(o._s1),
           "v": stats(o._s2)}
    hp = ctypes.byref(o._hp)
    for name in ("k2", "k3"):
        w, s1, s2, out = f.data.clone(), o._s1.clone(), o._s2.clone(), torch.empty_like(f.data)
        ts = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            if name == "k2":
                rc = lib.po_step(hp, w.data_ptr(), f.grad.data_ptr(), s1.data_ptr(), s2.data_ptr(), None, w.numel(),
                                 1e-4, o.step_count, None, None, torch.cuda.current_stream().cuda_stream)
            else:
                rc = lib.po_step_predict(hp, w.data_ptr(), f.grad.data_ptr(), s1.data_ptr(), s2.data_ptr(),
                                         out.data_ptr(), w.numel(), 1e-4, 3e-4, o.step_count, None, None,
                                         torch.cuda.current_stream().cuda_stream)
            e1.record()
            torch.cuda.synchronize()
            _lib.check(rc, name)
            ts.append(round(e0.elapsed_time(e1) * 1e3, 1))
        rep[name + "_us"] = ts
    print(json.dumps(rep), flush=True)
