"""Module stages (configs 2-4): weight-view semantics, partitioning, model
sizes. CPU only — no kernel launches."""

import itertools

import pytest
import torch
import torch.nn as nn

from paper_2312_00839_b200.stage_models import (
    LiveLinear,
    ModuleStage,
    balanced_partition,
    block_param_counts,
    build_module_stages,
    gnmt8_blocks,
    resnet101_blocks,
    vgg16_cifar_blocks,
)


def _predicted_views(stage, delta):
    hat = stage.flat.data.clone() + delta
    return hat, stage.flat.layout.views(hat)


def test_linear_backward_uses_live_weights_s9():
    torch.manual_seed(0)
    st = ModuleStage(1, [LiveLinear(3, 5)], "cpu", (3,))
    hat, hat_views = _predicted_views(st, 0.25)
    live_w = st.params[0].clone()
    x = torch.randn(4, 3)
    out = st.run_forward(hat_views, (1, 0), x, 1, check_finite=True)
    # forward used W_hat
    assert torch.allclose(out, x @ hat_views[0].t() + hat_views[1])
    g = torch.randn(4, 5)
    g_in, grads = st.run_backward(st.params, (1, 0), g)
    assert torch.allclose(g_in, g @ live_w)          # input grad with LIVE weights
    assert torch.allclose(grads[0], g.t() @ x)        # dW from the stashed input
    assert torch.allclose(grads[1], g.sum(0))
    assert torch.equal(st.params[0], live_w)          # prediction never wrote live weights


def test_conv_backward_uses_live_weights_s9():
    torch.manual_seed(1)
    st = ModuleStage(1, [nn.Conv2d(3, 4, 3, padding=1, bias=False)], "cpu", (3, 6, 6))
    hat, hat_views = _predicted_views(st, 0.1)
    live_w = st.params[0].clone()
    x = torch.randn(2, 3, 6, 6)
    out = st.run_forward(hat_views, (1, 0), x, 1)
    g = torch.randn_like(out)
    g_in, grads = st.run_backward(st.params, (1, 0), g)
    assert torch.allclose(g_in, torch.nn.grad.conv2d_input(x.shape, live_w, g, padding=1), atol=1e-5)
    assert torch.allclose(grads[0], torch.nn.grad.conv2d_weight(x, live_w.shape, g, padding=1), atol=1e-5)


def test_grads_overwrite_not_accumulate_and_flat_views():
    st = ModuleStage(1, [LiveLinear(3, 2)], "cpu", (3,))
    x = torch.randn(4, 3)
    for mb in (1, 2):
        out = st.run_forward(st.params, (mb, 0), x, mb)
        st.run_backward(st.params, (mb, 0), torch.ones_like(out))
    assert torch.allclose(st.flat.grads[0], torch.ones(4, 2).t() @ x)
    for p, v in zip(st.module.parameters(), st.params):
        assert p.data_ptr() == v.data_ptr()


def test_balanced_partition_is_optimal():
    costs = [5, 1, 1, 7, 2, 2, 9, 1, 3]
    for depth in range(1, len(costs) + 1):
        got = balanced_partition(costs, depth)
        assert got[0][0] == 0 and got[-1][1] == len(costs)
        assert all(a[1] == b[0] for a, b in zip(got, got[1:]))
        worst = max(sum(costs[a:b]) for a, b in got)
        best = min(
            max(sum(costs[a:b]) for a, b in zip((0,) + cuts, cuts + (len(costs),)))
            for cuts in itertools.combinations(range(1, len(costs)), depth - 1)
        )
        assert worst == best
    with pytest.raises(ValueError):
        balanced_partition([1, 2], 3)


def test_model_sizes_match_survey():
    assert abs(sum(block_param_counts(vgg16_cifar_blocks(100))) - 15.3e6) < 0.1e6
    assert abs(sum(block_param_counts(resnet101_blocks(200))) - 42.9e6) < 0.1e6
    assert sum(block_param_counts(gnmt8_blocks(1000, 64))) > 0


def test_vgg_stages_chain_shapes():
    stages = build_module_stages(vgg16_cifar_blocks(10), 4, "cpu", (3, 32, 32))
    assert [s.rank for s in stages] == [0, 1, 2, 3]
    for a, b in zip(stages, stages[1:]):
        assert a.out_shape == b.in_shape
    assert stages[-1].out_shape == (10,)
    x = torch.randn(2, 3, 32, 32)
    for st in stages:
        x = st.run_forward(st.params, (1, 0), x, 1)
    assert x.shape == (2, 10)
