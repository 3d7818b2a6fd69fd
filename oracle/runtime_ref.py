"""float64 restatement of the reference's dense-MLP stages and its
strategy-aware executor for the PipeOptim path — TEST ORACLE ONLY.

Follows pkg/src/pipesim:
  * stage math: affine + activation per layer, stash (inputs, pre-acts),
    backward dpre = g * act'(pre), dW = x^T dpre, db = colsum(dpre),
    g_in = dpre W_view^T with the BACKWARD-time view (stages.py:156-209,
    linalg.py:175-241). Transposes are materialised contiguously as
    Matrix.transpose does (linalg.py:60-61) so BLAS sees the same operands.
  * executor: events in timeline order (runtime.py:404-466) with the live
    policy (async_raw / serial / naive / gpipe) or the predictive policy
    (optimizer_prediction / spectrain: non-last stages forward on
    W - lr*s*dir, s the timeline-exact update gap; runtime.py:235-267).

Returns losses, version records, snapshot/stash peaks, final versions and
final parameters, all as plain Python / numpy values.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import schedule_ref
from .optim_ref import Hyper, OracleOptimizer, predict_weights


class OracleNumeric(RuntimeError):
    pass


def _act(pre, kind):
    if kind == "tanh":
        return np.tanh(pre)
    if kind == "relu":
        return np.maximum(pre, 0.0)
    return pre.copy()


def _act_grad(pre, kind):
    if kind == "tanh":
        t = np.tanh(pre)
        return 1.0 - t * t
    if kind == "relu":
        return (pre > 0.0).astype(pre.dtype)
    return np.ones_like(pre)


def _T(a):
    return np.ascontiguousarray(a.T)


def loss_and_grad(pred, target, kind):
    if kind == "mse":
        diff = pred - target
        n = diff.size
        return float(np.sum(diff * diff) / n), 2.0 * diff / n
    z = pred - pred.max(axis=1, keepdims=True)
    ez = np.exp(z)
    sm = ez / ez.sum(axis=1, keepdims=True)
    loss = float(np.mean(-np.log(np.sum(sm * target, axis=1))))
    return loss, (sm - target) / pred.shape[0]


def partition(n_layers: int, depth: int) -> list[list[int]]:
    q, r = divmod(n_layers, depth)
    out, lo = [], 0
    for k in range(depth):
        hi = lo + q + (1 if k < r else 0)
        out.append(list(range(lo, hi)))
        lo = hi
    return out


@dataclass
class Rec:
    mb: int
    stage: int
    forward_version: int
    predicted: bool
    prediction_target: int | None
    backward_version: int | None = None
    live_backward_version: int | None = None

    def as_tuple(self):
        return (self.mb, 0, self.stage, self.forward_version, self.predicted, self.prediction_target,
                self.backward_version, self.live_backward_version)


class _Stage:
    def __init__(self, rank, layer_ids, dims, acts, init, dtype=np.float64):
        self.rank = rank
        self.layer_ids = layer_ids
        self.acts = [acts[i] for i in layer_ids]
        self.params = []
        self.names = []
        for i in layer_ids:
            w, b = init(i, dims[i], dims[i + 1])
            self.params += [np.array(w, dtype=dtype), np.array(b, dtype=dtype)]
            self.names += [f"layer{i}.w", f"layer{i}.b"]
        self.version = 1
        self.stash = {}
        self.stash_peak = 0

    def forward(self, weights, key, x):
        ins, pres, h = [], [], x
        for j, kind in enumerate(self.acts):
            ins.append(h)
            pre = (h @ weights[2 * j]) + weights[2 * j + 1]
            pres.append(pre)
            h = _act(pre, kind)
        if not np.isfinite(h).all():
            raise OracleNumeric(f"non-finite value in stage {self.rank} forward output")
        self.stash[key] = (ins, pres)
        self.stash_peak = max(self.stash_peak, len(self.stash))
        return h

    def backward(self, weights, key, g):
        ins, pres = self.stash.pop(key)
        pg = [None] * len(weights)
        for j in reversed(range(len(self.acts))):
            dpre = g * _act_grad(pres[j], self.acts[j])
            pg[2 * j] = _T(ins[j]) @ dpre
            pg[2 * j + 1] = dpre.sum(axis=0, keepdims=True)
            g = dpre @ _T(weights[2 * j])
        return g, pg


def run(dims, acts, depth, n_batches, strategy, opt_hyper: Hyper, batch_fn, loss_kind, lr_for_mb,
        init, dtype=np.float64):
    """Execute a 1F1B (or serial, depth 1) run. `init(i, din, dout)` -> (w, b);
    `batch_fn(mb)` -> (x, y). Strategies: async_raw, optimizer_prediction,
    spectrain, serial. dtype=float64 is the reference; dtype=float32
    evaluates the same algorithm in fp32 (used only to size fp32 drift)."""
    if strategy == "serial" and depth != 1:
        raise ValueError("serial requires depth 1")
    predictive = strategy in ("optimizer_prediction", "spectrain")
    if strategy == "spectrain" and opt_hyper.kind != "sgdm":
        raise ValueError("spectrain requires the sgdm optimizer")
    groups = partition(len(dims) - 1, depth)
    stages = [_Stage(k, ids, dims, acts, init, dtype) for k, ids in enumerate(groups)]
    opts = [OracleOptimizer(opt_hyper, s.names) for s in stages]
    gap = schedule_ref.gaps(depth, n_batches)
    order = schedule_ref.global_order(depth, n_batches)

    acts_q, grads_q, cache = {}, {}, {}
    losses = [None] * n_batches
    records, rec_by = [], {}
    pending = [None] * depth
    predicting = set()
    snap = [1] * depth

    def batch(mb):
        if mb not in cache:
            x, y = batch_fn(mb)
            cache[mb] = (np.asarray(x, dtype=dtype), np.asarray(y, dtype=dtype))
        return cache[mb]

    for _slot, k, kind, mb in order:
        st, opt = stages[k], opts[k]
        if kind == schedule_ref.F:
            x = batch(mb)[0] if k == 0 else acts_q.pop((mb, k))
            lr = lr_for_mb(mb)
            predicting.discard(k)
            if predictive and k != depth - 1:
                s = gap[(mb, k)]
                view = predict_weights(st.params, lr, s, opt.prediction_direction(st.params))
                rec = Rec(mb, k, st.version, True, st.version + s)
                predicting.add(k)
            else:
                view = st.params
                rec = Rec(mb, k, st.version, False, None)
            try:
                out = st.forward(view, mb, x)
            except OracleNumeric as err:
                raise OracleNumeric(f"mb {mb} stage {k}: {err}") from err
            records.append(rec)
            rec_by[(mb, k)] = rec
            if k < depth - 1:
                acts_q[(mb, k + 1)] = out
            else:
                loss, g = loss_and_grad(out, batch(mb)[1], loss_kind)
                if not np.isfinite(loss):
                    raise OracleNumeric(f"mb {mb} stage {k}: non-finite loss under {loss_kind}")
                losses[mb - 1] = loss
                grads_q[(mb, k)] = g
        elif kind == schedule_ref.B:
            g_in, pg = st.backward(st.params, mb, grads_q.pop((mb, k)))
            if k > 0:
                grads_q[(mb, k - 1)] = g_in
            pending[k] = [p.copy() for p in pg]
            rec = rec_by[(mb, k)]
            rec.backward_version = st.version
            rec.live_backward_version = st.version
        else:
            try:
                st.params, _ = opt.step(st.params, pending[k], lr_for_mb(mb))
            except RuntimeError as err:
                raise OracleNumeric(f"mb {mb} stage {k}: {err}") from err
            st.version += 1
            pending[k] = None
        snap[k] = max(snap[k], 2 if k in predicting else 1)

    return dict(
        losses=losses,
        records=[r.as_tuple() for r in records],
        snapshot_peaks=snap,
        stash_peaks=[s.stash_peak for s in stages],
        final_versions=[s.version for s in stages],
        params=[[p.copy() for p in s.params] for s in stages],
        names=[list(s.names) for s in stages],
    )
