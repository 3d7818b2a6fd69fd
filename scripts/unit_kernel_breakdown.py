"""Where a config-1 stage unit's time goes: each stage's 16-unit CUDA graph
(bench_pipeline._unit_graph, the projection's unit) replayed under the torch
profiler (CUPTI kernel records, warm L2, clocks uncontrolled) — per kernel
family the device time per unit, plus the idle gaps between consecutive
kernels of the replay.

  python scripts/unit_kernel_breakdown.py [--stages 0,1] [--fuse-wgrad]
"""
import argparse
import collections
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2312_00839_b200 import bench_pipeline as bp  # noqa: E402
from paper_2312_00839_b200 import stages as S  # noqa: E402
from paper_2312_00839_b200.optim import OptimizerConfig, OptimizerState  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--stages", default="0,1,3")
ap.add_argument("--fuse-wgrad", action="store_true")
ap.add_argument("--replays", type=int, default=4)
a = ap.parse_args()
S.FUSE_WGRAD_UPDATE = a.fuse_wgrad
torch.backends.cuda.matmul.allow_tf32 = False
dev = torch.device("cuda", 0)
data = bp.DeviceBatches(torch, dev)
units = bp.UNITS_PER_GRAPH


def family(name: str) -> str:
    n = name
    for key, lab in (("GemmUniversal", "gemm_cutlass"), ("gemm", "gemm_other"), ("po_stream_kernel", "K1/K2/K3"),
                     ("splitk_bias_act", "splitk_bias_act"), ("relu_bwd_bias", "relu_bwd_bias"),
                     ("head_fwd", "head_fwd"), ("head_bwd", "head_bwd"), ("loss_grad", "loss_grad"),
                     ("all_finite", "all_finite"), ("wgrad_update", "wgrad_update(fused)"), ("Kernel", "other")):
        if key in n:
            return lab
    return n[:40]


for k in [int(s) for s in a.stages.split(",")]:
    for mode in ("pred_off", "pred_on"):
        st = S.build_stages(S.build_layers(bp.CONFIG1_DIMS, bp.CONFIG1_ACTS), 4, S.torch_init(7, dev), device=dev)
        opt = OptimizerState(OptimizerConfig("adam"), st[k].param_names, device=dev)
        g = bp._unit_graph(torch, dev, k, st[k], opt, data, "softmax_xent", mode == "pred_on", 4, units)
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.replays):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        unit_us = e0.elapsed_time(e1) * 1e3 / (a.replays * units)
        with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
            for _ in range(a.replays):
                g.replay()
            torch.cuda.synchronize()
        ev = sorted((e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA
                     and e.name and "Memcpy" not in e.name and "Memset" not in e.name),
                    key=lambda e: e.time_range.start)
        fam = collections.defaultdict(float)
        cnt = collections.Counter()
        gaps = 0.0
        prev_end = None
        for e in ev:
            f = family(e.name)
            fam[f] += e.time_range.elapsed_us()
            cnt[f] += 1
            if prev_end is not None and e.time_range.start > prev_end:
                gaps += e.time_range.start - prev_end
            prev_end = max(prev_end or 0, e.time_range.end)
        per = a.replays * units
        span = (ev[-1].time_range.end - ev[0].time_range.start) / per if ev else 0.0
        print(json.dumps({"stage": k, "mode": mode, "fuse_wgrad": a.fuse_wgrad, "unit_us_events": round(unit_us, 2),
                          "unit_us_profiled_span": round(span, 2), "gap_us_per_unit": round(gaps / per, 2),
                          "kernels_per_unit": round(len(ev) / per, 2),
                          "families_us_per_unit": {f: round(v / per, 2) for f, v in sorted(fam.items(),
                                                                                           key=lambda x: -x[1])},
                          "launches_per_unit": {f: round(c / per, 2) for f, c in cnt.items()}}), flush=True)
        del g, st, opt
        torch.cuda.empty_cache()
