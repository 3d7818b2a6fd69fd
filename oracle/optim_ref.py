"""numpy float64 restatement of the reference optimizer rules and the
optimizer-dependent predictor (pkg/src/pipesim/optim.py). TEST ORACLE ONLY.

Arithmetic is evaluated in the same order as the reference so that, on
identical float64 inputs, results are bit-identical to it (checked against the
reference's FROZEN_* golden trajectories and against fixtures generated from
the reference itself).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

KINDS = ("sgdm", "adam", "adamw")  # optim.py:17


class OracleNumericError(RuntimeError):
    pass


@dataclass(frozen=True)
class Hyper:
    """optim.py:20-43 defaults and range checks."""

    kind: str
    momentum: float = 0.9
    dampening: float = 0.0
    weight_decay: float = 5e-4
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    decoupled_decay: float = 1e-2

    def __post_init__(self):
        if self.kind not in KINDS:
            raise ValueError(f"unknown optimizer kind: {self.kind!r}")
        checks = [
            (0.0 <= self.momentum < 1.0, "momentum"),
            (0.0 <= self.dampening <= 1.0, "dampening"),
            (0.0 <= self.beta1 < 1.0, "beta1"),
            (0.0 <= self.beta2 < 1.0, "beta2"),
            (self.eps > 0.0, "eps"),
        ]
        for ok, name in checks:
            if not ok:
                raise ValueError(f"{name} out of range")


def bias_corrections(h: Hyper, t: int) -> tuple[float, float]:
    """1 - beta^t in Python float arithmetic (optim.py:106-108, :136-138)."""
    return 1.0 - h.beta1 ** t, 1.0 - h.beta2 ** t


def adam_ratio(m: np.ndarray, v: np.ndarray, bc1: float, bc2: float, eps: float) -> np.ndarray:
    """(m/bc1) / (sqrt(v/bc2) + eps)   (optim.py:115, :141)."""
    return (m / bc1) / (np.sqrt(v / bc2) + eps)


@dataclass
class OracleOptimizer:
    """Per-stage state over a list of float64 arrays (optim.py:46-59)."""

    hyper: Hyper
    names: list
    step_count: int = 0
    buf: list | None = None       # sgdm momentum buffer
    m: list | None = None         # adam exp_avg
    v: list | None = None         # adam exp_avg_sq

    def _directions(self, params, grads):
        h = self.hyper
        if h.kind == "sgdm":  # optim.py:89-99
            if self.buf is None:
                self.buf = [np.zeros_like(p) for p in params]
            out = []
            for i, (w, g) in enumerate(zip(params, grads)):
                eff = g + h.weight_decay * w
                nb = h.momentum * self.buf[i] + (1.0 - h.dampening) * eff
                self.buf[i] = nb
                out.append(nb.copy())
            return out
        if self.m is None:  # optim.py:101-119
            self.m = [np.zeros_like(p) for p in params]
            self.v = [np.zeros_like(p) for p in params]
        bc1, bc2 = bias_corrections(h, self.step_count + 1)
        out = []
        for i, (w, g) in enumerate(zip(params, grads)):
            m = h.beta1 * self.m[i] + (1.0 - h.beta1) * g
            v = h.beta2 * self.v[i] + (1.0 - h.beta2) * (g * g)
            self.m[i], self.v[i] = m, v
            d = adam_ratio(m, v, bc1, bc2, h.eps)
            if h.kind == "adamw":
                d = d + h.decoupled_decay * w
            out.append(d)
        return out

    def step(self, params, grads, lr):
        """optim.py:63-87: returns (new params, applied directions)."""
        if not (len(params) == len(grads) == len(self.names)):
            raise ValueError("step: params/grads/names length mismatch")
        dirs = self._directions(params, grads)
        new = []
        for name, w, d in zip(self.names, params, dirs):
            nw = w - lr * d
            if not np.isfinite(nw).all():
                raise OracleNumericError(f"optimizer step produced non-finite values in {name}")
            new.append(nw)
        self.step_count += 1
        return new, dirs

    def prediction_direction(self, params):
        """optim.py:123-142 (pure read; zeros before the first step; no lambda*W)."""
        if self.step_count == 0:
            return [np.zeros_like(p) for p in params]
        h = self.hyper
        if h.kind == "sgdm":
            return [b.copy() for b in self.buf]
        bc1, bc2 = bias_corrections(h, self.step_count)
        return [adam_ratio(m, v, bc1, bc2, h.eps) for m, v in zip(self.m, self.v)]


def predict_weights(params, lr, steps_ahead, directions):
    """Eq. (5), optim.py:145-155: w - (lr*s)*d."""
    if steps_ahead < 0:
        raise ValueError(f"steps_ahead must be >= 0, got {steps_ahead}")
    if len(params) != len(directions):
        raise ValueError("predict_weights: length mismatch")
    c = lr * steps_ahead
    return [w - c * d for w, d in zip(params, directions)]


def version_difference(depth: int, rank: int) -> int:
    """Eq. (4), optim.py:158-167."""
    if depth < 1:
        raise ValueError("depth must be >= 1")
    if not 0 <= rank < depth:
        raise ValueError("rank out of range")
    return depth - rank - 1


# ---- flat single-array helpers used by the parity tests and the CPU baseline ---


def flat_step(kind, w, g, s1, s2, lr, step_count, hyper: Hyper | None = None):
    """One K2 on flat float64 arrays; returns (w', s1', s2', d)."""
    h = hyper or Hyper(kind)
    st = OracleOptimizer(h, ["w"], step_count=step_count)
    if kind == "sgdm":
        st.buf = [s1.copy()]
    else:
        st.m, st.v = [s1.copy()], [s2.copy()]
    (nw,), (d,) = st.step([w], [g], lr)
    if kind == "sgdm":
        return nw, st.buf[0], None, d
    return nw, st.m[0], st.v[0], d


def flat_predict(kind, w, s1, s2, lr, steps_ahead, step_count, hyper: Hyper | None = None):
    """K1 on flat arrays: predict_weights(prediction_direction(...))."""
    h = hyper or Hyper(kind)
    st = OracleOptimizer(h, ["w"], step_count=step_count)
    if kind == "sgdm":
        st.buf = [s1]
    else:
        st.m, st.v = [s1], [s2]
    (d,) = st.prediction_direction([w])
    (wh,) = predict_weights([w], lr, steps_ahead, [d])
    return wh


def flat_step_predict(kind, w, g, s1, s2, lr, lr_pred, steps_ahead, step_count, hyper=None):
    """K3 = K2 then K1 on the updated state; returns (w', s1', s2', w_hat)."""
    nw, ns1, ns2, _ = flat_step(kind, w, g, s1, s2, lr, step_count, hyper)
    wh = flat_predict(kind, nw, ns1, ns2, lr_pred, steps_ahead, step_count + 1, hyper)
    return nw, ns1, ns2, wh


def inf_norm_rel(a: np.ndarray, b: np.ndarray) -> float:
    """max|a-b| / max|b| — the parity metric of SURVEY.md §8c (S15)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    den = float(np.max(np.abs(b), initial=0.0))
    num = float(np.max(np.abs(a - b), initial=0.0))
    if den == 0.0:
        return num
    return num / den


def algorithmic_bytes_per_param(kernel: str, kind: str) -> int:
    """SURVEY.md §8d table (fp32)."""
    sg = kind == "sgdm"
    return {
        "predict": 12 if sg else 16,
        "step": 20 if sg else 28,
        "step_predict": 24 if sg else 32,
    }[kernel]


__all__ = [
    "Hyper",
    "OracleOptimizer",
    "OracleNumericError",
    "predict_weights",
    "version_difference",
    "flat_step",
    "flat_predict",
    "flat_step_predict",
    "inf_norm_rel",
    "algorithmic_bytes_per_param",
    "bias_corrections",
    "adam_ratio",
]
