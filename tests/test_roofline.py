"""Counted-work pipeline bounds (roofline.py) on CPU stages: FLOPs and bytes
of config 1 by hand, and the bound structure."""

import pytest

from paper_2312_00839_b200 import roofline
from paper_2312_00839_b200.stages import build_layers, build_stages, torch_init


@pytest.fixture(scope="module")
def config1_stages():
    import torch

    dims, acts = [3072, 1024, 1024, 1024, 10], ["relu", "relu", "relu", "linear"]
    return build_stages(build_layers(dims, acts), 4, torch_init(0, torch.device("cpu")), device="cpu")


def test_config1_flops_and_bytes(config1_stages):
    B = 128
    st = config1_stages
    # stage 0: x@W forward + x^T dpre weight gradient (no input gradient)
    assert roofline.mlp_stage_flops(st[0], B) == 2 * (2 * B * 3072 * 1024)
    assert roofline.mlp_stage_flops(st[1], B) == 3 * (2 * B * 1024 * 1024)
    b = roofline.mlp_pipeline_bounds(st, B, 64, "adam", True, "fast_fp32")
    n0 = st[0].flat.layout.numel
    # W fwd + dW + K3 (32 B) + boundary in (x) / out (act + grad), both directions
    assert b["per_stage"][0]["mbytes"] == pytest.approx((4 * n0 + 4 * n0 + 32 * n0 + 2 * 4 * B * 3072
                                                         + 2 * 4 * B * 1024) / 1e6, abs=0.01)
    last = st[-1].flat.layout.numel
    off = roofline.mlp_pipeline_bounds(st, B, 64, "adam", False, "fast_fp32")
    assert off["per_stage"][-1]["mbytes"] == b["per_stage"][-1]["mbytes"]  # the last stage never fuses (K2)
    assert off["per_stage"][0]["mbytes"] < b["per_stage"][0]["mbytes"]  # K3 writes W_hat: +4 B/param
    assert off["per_stage"][-1]["mbytes"] * 1e6 >= 3 * 4 * last + 28 * last


def test_bounds_are_consistent(config1_stages):
    B, n = 128, 64
    b = roofline.mlp_pipeline_bounds(config1_stages, B, n, "adam", True, "fast_fp32")
    per = b["per_stage"]
    worst = max(max(p["compute_us"], p["hbm_us"]) for p in per) * 1e-6
    assert b["one_stage_per_gpu"]["samples_per_s"] == pytest.approx(B / worst * n / (n + 3), rel=1e-3)
    tot = max(sum(p["compute_us"] for p in per), sum(p["hbm_us"] for p in per)) * 1e-6
    assert b["single_gpu"]["samples_per_s"] == pytest.approx(B / tot, rel=1e-3)
    # config 1 is HBM-bound everywhere (optimizer pass >> GEMM time at fast-FP32 rates)
    assert b["single_gpu"]["bound"] == "hbm" and b["one_stage_per_gpu"]["bound"] == "hbm"
    assert b["one_stage_per_gpu"]["samples_per_s"] > b["single_gpu"]["samples_per_s"]
    pk = roofline.peaks()
    assert pk["tflops"]["fast_fp32"] == pytest.approx(pk["bf16_tflops"] / 3)
