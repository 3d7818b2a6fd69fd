"""Configs 2-4 (VGG-16 / ResNet-101 / GNMT-8) through the single-GPU 1F1B
runner: samples/s with prediction on vs off. Prints one JSON line per config."""
import argparse
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2312_00839_b200.bench_pipeline import MODULE_CONFIGS, single_gpu_module_pipeline  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default=",".join(MODULE_CONFIGS))
ap.add_argument("--n-batches", type=int, default=16)
ap.add_argument("--fp32", action="store_true")
ap.add_argument("--amp", default=None, choices=[None, "bf16"])
ap.add_argument("--no-eager", action="store_true")
ap.add_argument("--no-roofline", action="store_true")
a = ap.parse_args()
dev = torch.device("cuda", 0)
for name in a.configs.split(","):
    try:
        r = single_gpu_module_pipeline(torch, dev, name, n_batches=a.n_batches, tf32=not a.fp32, amp=a.amp,
                                       with_eager=not a.no_eager, with_roofline=not a.no_roofline)
    except Exception as exc:
        import traceback
        traceback.print_exc()
        r = {"error": f"{type(exc).__name__}: {exc}"}
    print(json.dumps({"config": name, **r}), flush=True)
    torch.cuda.empty_cache()
