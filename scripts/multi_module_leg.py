"""Dry run of one config's multi-rank module-pipeline leg (torchrun; gloo and
--share-gpu put every rank on cuda:0)."""
import json
import os
import sys
from pathlib import Path

import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2312_00839_b200.pipeline import bench_module_pipeline  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dist.init_process_group("gloo")
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
out = bench_module_pipeline(torch, dist, rank, world, dev, sys.argv[1], n_batches=int(sys.argv[2]), host_staging=True)
if rank == 0:
    print(json.dumps(out), flush=True)
dist.destroy_process_group()
