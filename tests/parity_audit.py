"""Per-update parity audit of real 1F1B runs (test infrastructure).

Installed as `paper_2312_00839_b200.optim.AUDIT`, it sees every eager K1 / K2
/ K3 launch of the run's OptimizerStates and every forward's weights, and
checks, launch by launch (BASELINE.json north_star: "predicted weights and
updated weights must match within 1e-6 relative in fp32"):

  * numerics — the launch's outputs (W', state', W_hat) against
      - the fp32 emulation of the kernels' documented evaluation order
        (oracle/optim_f32.py): bit-exact, and
      - the float64 reference rules (oracle/optim_ref.py, which restates
        /root/reference/pkg/src/pipesim/optim.py:63-155) evaluated on the
        same fp32 inputs: per parameter tensor max|a-b| / max|b| <= 1e-6
        (tensors of < 64 elements <= 1e-5, where the metric
        degenerates to elementwise);
  * the chain — each launch's inputs (W, state) are the previous launch's
    outputs (nothing else touched them), and every forward consumed exactly
    the W_hat the latest prediction produced (predicted forwards) or the
    live weights (runtime.py:242-258, S9/S10);
  * the coefficient plumbing — the logical sequence of updates and
    predictions per stage, with their learning rates, gaps and step counts,
    equals the one derived independently from the 1F1B rule
    (oracle/schedule_ref.py): U_j is step(lr_for_mb(j), t = updates so far),
    a predicted F_m is predict(lr_for_mb(m) [S4], s = gap(m, k), t = updates
    so far [S5]) (runtime.py:411-413, 449-463).

`check_tape` applies the plumbing check to a CUDA-graph replay: the device
coefficient slots a `CoefTape` refreshed must equal those of the expected
sequence at the replay's step counts and learning rates.
"""

from __future__ import annotations

import ctypes

import numpy as np

from oracle import optim_f32, optim_ref, schedule_ref

F32_TOL, SMALL_TOL, SMALL_N = 1e-6, 1e-5, 64


def _np(t):
    return None if t is None else t.detach().to("cpu").numpy().copy()


class ParityAudit:
    def __init__(self, stages, opts):
        self.stage_of = {id(o): k for k, o in enumerate(opts)}
        self.opts = list(opts)
        self.layouts = [s.flat.layout for s in stages]
        # (W, s1, s2) fp32 numpy: the live weights / state after the last launch
        self.state = [(_np(s.flat.data), _np(o._s1), _np(o._s2)) for s, o in zip(stages, opts)]
        self.what = [None] * len(opts)   # the last W_hat produced
        self.log = [[] for _ in opts]    # logical ops per stage
        self.launches = [[] for _ in opts]
        self.forwards = 0
        self.max_rel = {"w": 0.0, "state": 0.0, "w_hat": 0.0}

    # -- hooks ------------------------------------------------------------------
    def before(self, opt, op, flat, out):
        import torch

        torch.cuda.synchronize()
        k = self.stage_of[id(opt)]
        w = _np(flat.data)
        g = _np(flat.grad) if op != "predict" else None
        s1, s2 = _np(opt._s1), _np(opt._s2)
        pw, ps1, ps2 = self.state[k]  # nothing but our launches touches W / state
        assert np.array_equal(w, pw), f"stage {k}: live weights changed outside the optimizer"
        if ps1 is not None:
            assert np.array_equal(s1, ps1) and (ps2 is None or np.array_equal(s2, ps2)), \
                f"stage {k}: optimizer state changed outside the optimizer"
        return (k, opt, op, flat, out, opt.step_count, w, g, s1, s2)

    def after(self, tok, lr, lr_pred, steps_ahead):
        import torch

        torch.cuda.synchronize()
        k, opt, op, flat, out, t, w, g, s1, s2 = tok
        kind = opt.config.kind
        hp = {f: getattr(opt.config, f) for f in ("momentum", "dampening", "weight_decay", "beta1", "beta2", "eps",
                                                   "decoupled_decay")}
        hyper = optim_ref.Hyper(kind, **hp)
        n = w.size
        z = np.zeros(n, np.float32)
        if s1 is None:  # lazily-zero state (optim.py:91-92, 103-105)
            s1 = z
        if s2 is None and kind != "sgdm":
            s2 = z
        d64 = lambda a: None if a is None else a.astype(np.float64)  # noqa: E731
        if op == "predict":
            c_pred = float(lr_pred) * steps_ahead
            wh = _np(out)
            want32 = optim_f32.predict(kind, w, s1, s2, c_pred, t, **hp)
            assert np.array_equal(wh, want32), f"stage {k}: K1 not bit-exact vs the fp32 emulation (t={t})"
            want64 = optim_ref.flat_predict(kind, d64(w), d64(s1), d64(s2), float(lr_pred), steps_ahead, t, hyper)
            self._rel(k, "w_hat", wh, want64)
            self.what[k] = wh
            self.log[k].append(("predict", float(lr_pred), int(steps_ahead), t))
        else:
            nw, ns1, ns2 = _np(flat.data), _np(opt._s1), _np(opt._s2)
            fused = op == "step_predict"
            c_pred = float(lr_pred) * steps_ahead if fused else None
            ew, es1, es2, ewh = optim_f32.step(kind, w, g, s1, s2, float(lr), t, c_pred=c_pred, **hp)
            assert np.array_equal(nw, ew), f"stage {k}: updated W not bit-exact vs the fp32 emulation (t={t})"
            assert np.array_equal(ns1, es1) and (es2 is None or np.array_equal(ns2, es2)), \
                f"stage {k}: updated state not bit-exact vs the fp32 emulation (t={t})"
            if fused:
                rw, rs1, rs2, rwh = optim_ref.flat_step_predict(kind, d64(w), d64(g), d64(s1), d64(s2), float(lr),
                                                                float(lr_pred), steps_ahead, t, hyper)
            else:
                rw, rs1, rs2, _ = optim_ref.flat_step(kind, d64(w), d64(g), d64(s1), d64(s2), float(lr), t, hyper)
            self._rel(k, "w", nw, rw)
            self._rel(k, "state", ns1, rs1)
            if rs2 is not None:
                self._rel(k, "state", ns2, rs2)
            self.log[k].append(("step", float(lr), t))
            if fused:
                wh = _np(out)
                assert np.array_equal(wh, ewh), f"stage {k}: K3 W_hat not bit-exact vs the fp32 emulation (t={t})"
                self._rel(k, "w_hat", wh, rwh)
                self.what[k] = wh
                self.log[k].append(("predict", float(lr_pred), int(steps_ahead), t + 1))
            self.state[k] = (nw, ns1, ns2)
        self.launches[k].append(op)

    def forward(self, opt, mb, micro, weights, predicted):
        import torch

        k = self.stage_of[id(opt)]
        torch.cuda.synchronize()
        lay = self.layouts[k]
        got = np.zeros(lay.numel, np.float32)
        for o, n, v in zip(lay.offsets, lay.sizes, weights):
            got[o:o + n] = _np(v).reshape(-1)
        if predicted:
            assert self.what[k] is not None, f"stage {k}: predicted forward of mb {mb} before any prediction"
            assert np.array_equal(got, self.what[k]), f"stage {k}: forward of mb {mb} did not read the latest W_hat"
            last = self.log[k][-1]
            assert last[0] == "predict" and len(last) == 4, f"stage {k}: W_hat of mb {mb} consumed twice"
            self.log[k][-1] = last + (mb,)
        else:
            assert np.array_equal(got, self.state[k][0]), f"stage {k}: live forward of mb {mb} did not read the live weights"
        self.forwards += 1

    # -- checks -----------------------------------------------------------------
    def _rel(self, k, what, got, want):
        lay = self.layouts[k]
        for name, o, n in zip(lay.names, lay.offsets, lay.sizes):
            r = optim_ref.inf_norm_rel(got[o:o + n], want[o:o + n])
            tol = F32_TOL if n >= SMALL_N else SMALL_TOL
            assert r <= tol, f"stage {k} {what} {name}: {r:.3e} > {tol:g} vs the float64 reference"
            self.max_rel[what] = max(self.max_rel[what], r if n >= SMALL_N else 0.0)

    def check_sequence(self, depth, n_batches, lr_for_mb, predictive, fused=None):
        """The logged per-stage op sequence == the one the 1F1B rule implies."""
        for k in range(depth):
            want = expected_ops(depth, n_batches, k, lr_for_mb, predictive)
            got = self.log[k]
            assert got == want, f"stage {k}: op sequence differs\n got {got[:6]}...\nwant {want[:6]}..."
            if fused is not None and predictive and k < depth - 1:
                n_k3 = sum(1 for op in self.launches[k] if op == "step_predict")
                assert (n_k3 > 0) == fused

    def counts(self):
        return sum(len(x) for x in self.launches), self.forwards


def expected_ops(depth, n_batches, k, lr_for_mb, predictive, t0=0):
    """Stage k's logical optimizer ops from the 1F1B rule: ('step', lr, t) per
    update, ('predict', lr_pred, s, t, mb) per predicted forward."""
    gaps = schedule_ref.gaps(depth, n_batches)
    out, t = [], t0
    for kind, m in schedule_ref.stage_sequence(depth, n_batches, k):
        if kind == schedule_ref.U:
            out.append(("step", float(lr_for_mb(m)), t))
            t += 1
        elif kind == schedule_ref.F and predictive and k < depth - 1:
            out.append(("predict", float(lr_for_mb(m)), gaps[(m, k)], t, m))
    return out


def check_tape(tape, opts, depth, n_batches, lr_for_mb, predictive, step_counts):
    """After CoefTape.refresh (and a sync): every device coefficient slot ==
    po_coef_fill of the expected op at the replay's step counts."""
    import torch

    from paper_2312_00839_b200 import _lib

    torch.cuda.synchronize()
    dev = tape.dev[: 4 * len(tape.entries)].cpu().numpy().reshape(-1, 4)
    lib = _lib.load()
    by_opt = {id(o): [] for o in opts}
    for i, (opt, which, rel, lr, lr_pred, s) in enumerate(tape.entries):
        by_opt[id(opt)].append((i, which, rel, s))
    for k, o in enumerate(opts):
        want = expected_ops(depth, n_batches, k, lr_for_mb, predictive, t0=step_counts[k])
        got_ops, j = [], 0
        for i, which, rel, s in by_opt[id(o)]:
            ops = []
            if which in (_lib.PO_COEF_STEP, _lib.PO_COEF_STEP_PREDICT):
                ops.append(want[j])
                assert want[j][0] == "step", f"stage {k}: slot {i} is an update where the rule has {want[j]}"
                j += 1
            if which in (_lib.PO_COEF_PREDICT, _lib.PO_COEF_STEP_PREDICT):
                assert want[j][0] == "predict" and want[j][2] == s, f"stage {k}: slot {i} vs {want[j]}"
                ops.append(want[j])
                j += 1
            step = next((op for op in ops if op[0] == "step"), None)
            pred = next((op for op in ops if op[0] == "predict"), None)
            lr = step[1] if step else 0.0
            c = pred[1] * pred[2] if pred else 0.0
            t = step[2] if step else pred[3]
            if pred is not None and step is not None:
                assert pred[3] == step[2] + 1
            buf = _lib.po_coef()
            _lib.check(lib.po_coef_fill(ctypes.byref(o._hp), which, lr, c, t, ctypes.byref(buf)), "po_coef_fill")
            exp = np.array([buf.lr, buf.c_pred, buf.inv_bc1, buf.inv_bc2], np.float32)
            assert np.array_equal(dev[i], exp), f"stage {k}: tape slot {i} {dev[i]} != {exp} for {ops}"
            got_ops += ops
        assert got_ops == want, f"stage {k}: the graph's launches do not cover the rule's op sequence"
