"""Pipeline legs of bench.py: config 1 (4-stage 3072-1024^3-10 MLP, ReLU x3 +
linear, softmax cross-entropy, B = 128, Adam lr 1e-4) on synthetic
CIFAR-10-shaped batches resident in HBM, 1F1B with prediction on
(optimizer_prediction) vs off (async_raw, the prediction-disabled control).
"""

from __future__ import annotations

import time

CONFIG1_DIMS = [3072, 1024, 1024, 1024, 10]
CONFIG1_ACTS = ["relu", "relu", "relu", "linear"]
BATCH = 128


class DeviceBatches:
    """Synthetic x ~ N(0,1) (B, 3072) and one-hot labels uniform over 10,
    pre-generated on the device (inputs resident in HBM)."""

    def __init__(self, torch, device, n_distinct: int = 16, seed: int = 0, dims=CONFIG1_DIMS):
        g = torch.Generator(device=device).manual_seed(seed)
        self.x = [torch.randn(BATCH, dims[0], device=device, generator=g) for _ in range(n_distinct)]
        self.y = []
        for _ in range(n_distinct):
            lab = torch.randint(0, dims[-1], (BATCH,), device=device, generator=g)
            self.y.append(torch.nn.functional.one_hot(lab, dims[-1]).float())

    def batch(self, mb: int):
        i = (mb - 1) % len(self.x)
        return self.x[i], self.y[i]


def _run_once(torch, device, strategy, depth, n_batches, data, seed=0, dims=CONFIG1_DIMS, acts=CONFIG1_ACTS):
    from .optim import OptimizerConfig, OptimizerState
    from .runtime import build_timeline, execute
    from .stages import build_layers, build_stages, torch_init

    stages = build_stages(build_layers(dims, acts), depth, torch_init(seed, device), device=device)
    opts = [OptimizerState(OptimizerConfig("adam"), s.param_names, device=device) for s in stages]
    tl = build_timeline(strategy, depth, n_batches)
    torch.cuda.synchronize(device)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    rep = execute(tl, stages, opts, strategy, data, "softmax_xent", lambda mb: 1e-4, checks="deferred")
    e1.record()
    torch.cuda.synchronize(device)
    wall = time.perf_counter() - t0
    return rep, e0.elapsed_time(e1) / 1e3, wall


def single_gpu_pipeline(torch, device, n_batches: int = 64, depth: int = 4):
    """All `depth` stages on one GPU, events in timeline order (the single-GPU
    1F1B runner). Reports samples/s with prediction on and off."""
    torch.backends.cuda.matmul.allow_tf32 = False
    data = DeviceBatches(torch, device)
    out = {"config": f"config1 MLP {CONFIG1_DIMS}, B={BATCH}, Adam lr 1e-4, 1F1B D={depth} on 1 GPU "
                     f"(single-process runner), {n_batches} mini-batches, fp32 GEMMs (TF32 off)"}
    launches = 0
    for strategy in ("async_raw", "optimizer_prediction"):
        _run_once(torch, device, strategy, depth, min(n_batches, 2 * depth + 2), data)  # warm-up
        rep, sec, wall = _run_once(torch, device, strategy, depth, n_batches, data)
        key = "pred_on" if strategy == "optimizer_prediction" else "pred_off"
        out[key] = {"samples_per_s": round(n_batches * BATCH / sec, 1), "s": round(sec, 4),
                    "wall_s": round(wall, 4), "final_loss": rep.losses[-1]}
        # predictor/optimizer launches: one per update (K2/K3) + K1 per unfused predicted forward
        launches += n_batches * depth + (n_batches if strategy == "optimizer_prediction" else 0)
    on, off = out["pred_on"]["samples_per_s"], out["pred_off"]["samples_per_s"]
    out["value"] = on
    out["unit"] = "samples/s"
    out["prediction_overhead"] = round(1.0 - on / off, 4)
    out["launches"] = launches
    return out


def multi_gpu_pipeline(torch, dist, rank, world, device, n_batches: int = 64):
    """One stage per GPU over NCCL (pipeline.py); depth = world."""
    from .pipeline import bench_config1_pipeline

    return bench_config1_pipeline(torch, dist, rank, world, device, n_batches=n_batches)
