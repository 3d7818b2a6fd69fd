"""Config-1 single-GPU pipeline leg alone (stage-concurrent + serial runners,
prediction on/off), for iterating on the runner without the kernel leg."""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2312_00839_b200 import bench_pipeline as bp  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--tf32", action="store_true")
ap.add_argument("--n-batches", type=int, default=64)
ap.add_argument("--no-eager", action="store_true")
a = ap.parse_args()
dev = torch.device("cuda", 0)
r = bp.single_gpu_pipeline(torch, dev, n_batches=a.n_batches, tf32=a.tf32, with_eager=not a.no_eager)
print(json.dumps(r))
