"""float32 emulation of the kernels' documented arithmetic — TEST ORACLE ONLY.

The reference formulas (pkg/src/pipesim/optim.py:89-155, see optim_ref.py)
evaluated in numpy float32 with exactly the operation order the sm_100a
kernels use (csrc/pipeoptim_kernels.cu `elem`): every multiply/add/divide/sqrt
rounded separately to fp32 (the kernels use __fmul_rn/__fadd_rn/__fdiv_rn/
__fsqrt_rn, so no FMA contraction), coefficients derived in float64 and
rounded once. The kernels must match this BIT FOR BIT; optim_ref.py (float64,
bit-identical to the reference) bounds the fp32 rounding itself.
"""

from __future__ import annotations

import numpy as np

f32 = np.float32


def coef(kind, lr=0.0, c_pred=0.0, t=0, momentum=0.9, dampening=0.0, weight_decay=5e-4,
         beta1=0.9, beta2=0.999, eps=1e-8, decoupled_decay=1e-2):
    # reciprocal bias corrections, formed in double and rounded once
    ibc1 = 1.0 / (1.0 - beta1 ** t) if t >= 1 else 1.0
    ibc2 = 1.0 / (1.0 - beta2 ** t) if t >= 1 else 1.0
    return dict(
        lr=f32(lr), c=f32(c_pred), ibc1=f32(ibc1), ibc2=f32(ibc2), b1=f32(beta1), omb1=f32(1.0 - beta1),
        b2=f32(beta2), omb2=f32(1.0 - beta2), eps=f32(eps), lam=f32(decoupled_decay), mom=f32(momentum),
        omd=f32(1.0 - dampening), wd=f32(weight_decay),
    )


def _ratio(m, v, k):
    # the kernels' order: (m * ibc1) / (sqrt(v * ibc2) + eps) — the reference's
    # (m / bc1) / (sqrt(v / bc2) + eps) with the bias corrections applied as
    # correctly-rounded multiplies by their reciprocals
    return (m * k["ibc1"]) / (np.sqrt(v * k["ibc2"]) + k["eps"])


def step(kind, w, g, s1, s2, lr, step_count, c_pred=None, **hp):
    """K2 (c_pred None) or K3; returns (w', s1', s2', w_hat or None)."""
    k = coef(kind, lr, 0.0 if c_pred is None else c_pred, step_count + 1, **hp)
    w, g, s1 = w.astype(f32), g.astype(f32), s1.astype(f32)
    if kind == "sgdm":
        eff = g + k["wd"] * w
        nb = k["mom"] * s1 + k["omd"] * eff
        nw = w - k["lr"] * nb
        wh = None if c_pred is None else nw - k["c"] * nb
        return nw, nb, None, wh
    s2 = s2.astype(f32)
    m = k["b1"] * s1 + k["omb1"] * g
    v = k["b2"] * s2 + k["omb2"] * (g * g)
    r = _ratio(m, v, k)
    d = r + k["lam"] * w if kind == "adamw" else r
    nw = w - k["lr"] * d
    wh = None if c_pred is None else nw - k["c"] * r
    return nw, m, v, wh


def predict(kind, w, s1, s2, lr_times_s, step_count, **hp):
    k = coef(kind, 0.0, lr_times_s, step_count, **hp)
    w = w.astype(f32)
    if step_count == 0:
        return w - k["c"] * f32(0.0)
    if kind == "sgdm":
        return w - k["c"] * s1.astype(f32)
    return w - k["c"] * _ratio(s1.astype(f32), s2.astype(f32), k)
