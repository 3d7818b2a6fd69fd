"""Pipeline rooflines from counted work (BASELINE.json: "the
slower of stage compute and NVLink transfer for the pipeline").

For every stage k and one mini-batch, the stage unit (forward + backward +
update) is bounded below by three independent terms:

  compute  FLOPs_k / peak(arith)   dense GEMM/conv FLOPs of forward and
                                   backward (2·M·N·K per product; the weight
                                   and input gradients each cost a forward),
                                   at the peak of the arithmetic the stage
                                   actually runs: fast-FP32 (3 bf16 products
                                   per fp32 product on tcgen05) = bf16/3,
                                   TF32 = bf16/2, bf16 = bf16 (the sustained
                                   dense bf16 figure of MEASURED_PEAKS.json)
  hbm      bytes_k / hbm_gbs       compulsory bytes: the weights read by the
                                   forward and by the input gradient, the
                                   weight gradient written, the optimizer pass
                                   (K2 or K3 algorithmic bytes, 20-32 B/param)
                                   and the stage's boundary tensors (input and
                                   output activation, both gradients)
  link     boundary bytes / 900 GB/s per NVLink-5 direction (activation and
                                   gradient of a boundary travel in opposite
                                   directions)

One stage per GPU: the pipeline runs at most at B / max_k max(compute_k,
hbm_k) samples/s times the 1F1B fill/drain factor n / (n + D - 1)
(`schedule.py:356-386` makespan), and at most at B / max link time. All D
stages on ONE GPU (the single-GPU runners): the stages share its tensor
cores and HBM, so B / max(Σ_k compute_k, Σ_k hbm_k). Both are upper bounds
on throughput, so every measured fraction is <= 1 unless caches beat the
compulsory traffic (stated where it happens).
"""

from __future__ import annotations

import json
import math
from pathlib import Path

NVLINK_GBS = 900.0  # NVLink 5, per direction per GPU (B200_PROFILING.md)
FP32_SIMT_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12  # 74.4: FFMA peak at max SM clock

_PEAKS = Path(__file__).resolve().parent.parent / "MEASURED_PEAKS.json"


def peaks() -> dict:
    """Measured HBM copy GB/s and sustained dense bf16 TFLOP/s (driver-written
    MEASURED_PEAKS.json), else the B200_PROFILING.md fallbacks."""
    try:
        d = json.loads(_PEAKS.read_text())
        hbm, bf16 = float(d["hbm_gbs"]), float(d.get("bf16_tflops_sustained", d["bf16_tflops"]))
        src = "MEASURED_PEAKS.json (hbm_gbs, bf16_tflops_sustained)"
    except Exception:
        hbm, bf16, src = 6650.0, 1400.0, "B200_PROFILING.md fallback"
    return {"hbm_gbs": hbm, "bf16_tflops": bf16, "source": src,
            "tflops": {"fast_fp32": bf16 / 3, "tf32": bf16 / 2, "bf16": bf16, "fp32_simt": FP32_SIMT_TFLOPS}}


def opt_bytes_per_param(kind: str, fused: bool) -> int:
    """K2 20/28 B, K3 24/32 B per fp32 parameter."""
    sg = kind == "sgdm"
    return (24 if sg else 32) if fused else (20 if sg else 28)


def mlp_stage_flops(stage, batch: int) -> float:
    """Forward + backward GEMM FLOPs of one MLP stage (stages.py: per layer
    x@W forward, x^T·dpre weight gradient, dpre·W^T input gradient — the
    latter skipped for stage 0's first layer, whose input needs no gradient)."""
    f = 0.0
    for i, spec in enumerate(stage.layers):
        mnk = 2.0 * batch * spec.in_dim * spec.out_dim
        f += 2 * mnk if (stage.rank == 0 and i == 0) else 3 * mnk
    return f


def module_stage_flops(torch, stage, batch: int, in_dtype=None) -> float:
    """Forward + backward FLOPs of one module stage, counted by PyTorch's
    FlopCounterMode over one real forward + backward (convolutions, matmuls,
    and the LSTM's GEMMs; elementwise work is not counted)."""
    from torch.utils.flop_counter import FlopCounterMode

    dev = stage.flat.device
    shape = (batch, *stage.in_shape)
    if in_dtype is not None and not in_dtype.is_floating_point:
        x = torch.zeros(shape, dtype=torch.float32, device=dev)
    else:
        x = torch.randn(shape, device=dev)
    g = torch.randn((batch, *stage.out_shape), device=dev)
    with FlopCounterMode(display=False) as fc:
        stage.run_forward(stage.params, ("flops", 0), x, stage.version, check_finite=False)
        stage.run_backward(stage.params, ("flops", 0), g, need_input_grad=stage.rank > 0)
    stage.flat.grad.zero_()
    return float(fc.get_total_flops())


def stage_bytes(numel: int, kind: str, fused: bool, boundary_in: int, boundary_out: int, first: bool) -> int:
    """Compulsory HBM bytes of one stage unit: W read by the forward (W or
    W_hat) and by the input gradient (not on stage 0), dW written, the
    optimizer pass, and the boundary tensors in both directions."""
    w = 4 * numel
    params = w + (0 if first else w) + w + opt_bytes_per_param(kind, fused) * numel
    return params + 2 * boundary_in + 2 * boundary_out


def bounds(flops, bytes_, boundary_bytes, batch: int, n: int, depth: int, arith: str) -> dict:
    """Per-stage terms and the two pipeline bounds (samples/s)."""
    pk = peaks()
    tf = pk["tflops"][arith] * 1e12
    hbm = pk["hbm_gbs"] * 1e9
    comp = [f / tf for f in flops]
    mem = [b / hbm for b in bytes_]
    stage_t = [max(c, m) for c, m in zip(comp, mem)]
    link_t = max(boundary_bytes) / (NVLINK_GBS * 1e9) if boundary_bytes else 0.0
    fill = n / (n + depth - 1)
    per_gpu_compute = batch / max(stage_t) * fill
    per_gpu_link = batch / link_t if link_t else math.inf
    one_gpu_t = max(sum(comp), sum(mem))
    k_max = max(range(depth), key=lambda k: stage_t[k])
    return {
        "one_stage_per_gpu": {
            "samples_per_s": round(min(per_gpu_compute, per_gpu_link), 1),
            "bound": "link" if per_gpu_link < per_gpu_compute else
                     ("compute" if comp[k_max] >= mem[k_max] else "hbm"),
            "bottleneck_stage": k_max,
            "fill_drain_factor": round(fill, 4),
            "link_samples_per_s": None if math.isinf(per_gpu_link) else round(per_gpu_link, 1),
        },
        "single_gpu": {
            "samples_per_s": round(batch / one_gpu_t, 1),
            "bound": "compute" if sum(comp) >= sum(mem) else "hbm",
        },
        "per_stage": [{"gflop": round(f / 1e9, 3), "mbytes": round(b / 1e6, 2), "compute_us": round(c * 1e6, 2),
                       "hbm_us": round(m * 1e6, 2)} for f, b, c, m in zip(flops, bytes_, comp, mem)],
        "arith": arith,
        "peak_tflops": round(pk["tflops"][arith], 1),
        "peak_hbm_gbs": pk["hbm_gbs"],
        "link_gbs": NVLINK_GBS,
        "peak_source": pk["source"],
    }


def mlp_pipeline_bounds(stages, batch: int, n: int, kind: str, fused: bool, arith: str) -> dict:
    depth = len(stages)
    flops = [mlp_stage_flops(s, batch) for s in stages]
    bnd = [4 * batch * s.out_dim for s in stages[:-1]]
    bytes_ = []
    for k, s in enumerate(stages):
        b_in = 4 * batch * s.in_dim
        b_out = 4 * batch * s.out_dim if k < depth - 1 else 0
        bytes_.append(stage_bytes(s.flat.layout.numel, kind, fused and k < depth - 1, b_in, b_out, k == 0))
    return bounds(flops, bytes_, bnd, batch, n, depth, arith)


def module_pipeline_bounds(torch, stages, batch: int, n: int, kind: str, fused: bool, arith: str,
                           in_dtype=None) -> dict:
    depth = len(stages)
    flops = [module_stage_flops(torch, s, batch, in_dtype if k == 0 else None) for k, s in enumerate(stages)]
    bnd = [4 * batch * math.prod(s.out_shape) for s in stages[:-1]]
    bytes_ = []
    for k, s in enumerate(stages):
        b_in = 4 * batch * math.prod(s.in_shape)
        b_out = 4 * batch * math.prod(s.out_shape) if k < depth - 1 else 0
        bytes_.append(stage_bytes(s.flat.layout.numel, kind, fused and k < depth - 1, b_in, b_out, k == 0))
    return bounds(flops, bytes_, bnd, batch, n, depth, arith)
