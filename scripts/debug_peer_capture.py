"""Debug driver: config-1 peer runner capture on 2 ranks sharing one GPU,
reporting the stream capture status after every device call of the run."""
import ctypes
import os
import sys
from pathlib import Path

import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2312_00839_b200 import _lib  # noqa: E402
from paper_2312_00839_b200.bench_pipeline import BATCH, CONFIG1_ACTS, CONFIG1_DIMS, DeviceBatches  # noqa: E402
from paper_2312_00839_b200.peer_pipeline import bench_peer_pipeline  # noqa: E402
from paper_2312_00839_b200.stages import StageModel, build_layers, partition_layers, torch_init  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dist.init_process_group("gloo")
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
cudart = ctypes.CDLL("libcudart.so.12")
status = ctypes.c_int()


def cap_status():
    s = torch.cuda.current_stream().cuda_stream
    cudart.cudaStreamIsCapturing(ctypes.c_void_p(s), ctypes.byref(status))
    return status.value  # 0 none, 1 active, 2 invalidated


orig = _lib.check


def check(rc, what):
    st = cap_status()
    if st == 2:
        print(f"rank {rank}: capture invalidated at/before {what}", file=sys.stderr, flush=True)
    orig(rc, what)


_lib.check = check
if sys.argv[1:] == ["prior"]:
    from paper_2312_00839_b200.pipeline import bench_config1_pipeline
    print(bench_config1_pipeline(torch, dist, rank, world, dev, n_batches=16, host_staging=True), flush=True)
else:
    layers = build_layers(CONFIG1_DIMS, CONFIG1_ACTS)
    data = DeviceBatches(torch, dev)
    out = bench_peer_pipeline(torch, dist, rank, world, dev,
                              lambda: StageModel(rank, partition_layers(layers, world)[rank], torch_init(0, dev), dev),
                              data, "softmax_xent", 1e-4, BATCH, int(sys.argv[2]) if len(sys.argv) > 2 else 16)
    print(rank, out, flush=True)
dist.destroy_process_group()
