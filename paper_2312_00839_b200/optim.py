"""Optimizer rules and optimizer-dependent weight prediction on B200.

Drop-in for the reference's predictor interface (pkg/src/pipesim/optim.py):
`OptimizerConfig`, `OptimizerState(config, names)` with `.step(params, grads,
lr) -> (new_params, dirs)`, `.prediction_direction(params)`, `.step_count`,
`.momentum_buf / .exp_avg / .exp_avg_sq`, plus `predict_weights` and
`version_difference` — same names, argument meaning and errors.

What changes underneath: per-stage state lives in FLAT fp32 device buffers
(`FlatLayout`), and every arithmetic pass is one of the sm_100a kernels in
csrc/pipeoptim_kernels.cu called through the C-ABI (include/pipeoptim.h).
Besides the reference-shaped list API, the runtime uses the in-place fast
paths on a `FlatParams`:

  step_(flat, lr)                                   K2  (28 / 20 B per param)
  predict_(flat, lr, steps_ahead, out)              K1  (16 / 12 B per param)
  step_predict_(flat, lr, lr_pred, steps_ahead, out) K3 (32 / 24 B per param)

There is no CPU fallback: CPU tensors are accepted only as HOST buffers that
are staged through the device (the end-to-end path), and a missing
libpipeoptim.so raises `LibraryMissing`.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass
from typing import Sequence

import torch

from . import _lib
from .errors import NumericError

OPTIMIZER_KINDS = ("sgdm", "adam", "adamw")

_INT64_MAX = (1 << 63) - 1

# Test-only launch audit (tests/parity_audit.py). When set, every eager K1 /
# K2 / K3 launch of an OptimizerState is bracketed by AUDIT.before(opt, op,
# flat, out) -> token and AUDIT.after(token, lr, lr_pred, steps_ahead), and
# runtime.execute reports each forward's weights (AUDIT.forward), so a test
# can replay every update and prediction of a real run through the oracle.
# None in production: one attribute test per launch.
AUDIT = None


@dataclass(frozen=True)
class OptimizerConfig:
    """Validated hyper-parameters; defaults and ranges as optim.py:20-43."""

    kind: str
    momentum: float = 0.9
    dampening: float = 0.0
    weight_decay: float = 5e-4
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    decoupled_decay: float = 1e-2

    def __post_init__(self):
        if self.kind not in OPTIMIZER_KINDS:
            raise ValueError(f"unknown optimizer kind: {self.kind!r}")
        if not 0.0 <= self.momentum < 1.0:
            raise ValueError(f"momentum must be in [0, 1), got {self.momentum}")
        if not 0.0 <= self.dampening <= 1.0:
            raise ValueError(f"dampening must be in [0, 1], got {self.dampening}")
        for name in ("beta1", "beta2"):
            v = getattr(self, name)
            if not 0.0 <= v < 1.0:
                raise ValueError(f"{name} must be in [0, 1), got {v}")
        if self.eps <= 0.0:
            raise ValueError(f"eps must be positive, got {self.eps}")

    def hparams(self) -> _lib.po_hparams:
        return _lib.po_hparams(
            _lib.KIND_CODES[self.kind],
            0,
            float(self.momentum),
            float(self.dampening),
            float(self.weight_decay),
            float(self.beta1),
            float(self.beta2),
            float(self.eps),
            float(self.decoupled_decay),
        )


# ---- flat per-stage layout ----------------------------------------------------


class FlatLayout:
    """Parameters [w0, b0, w1, b1, ...] (stages.py:133-138) packed into one flat
    fp32 buffer. Each parameter starts on a 64-element (256 B) boundary so every
    view is aligned for the 256-bit vector path; padding stays zero under all
    three rules (g = 0, W = 0 => state and W remain 0).
    """

    ALIGN = 64

    def __init__(self, names: Sequence[str], shapes: Sequence[Sequence[int]]):
        if len(names) != len(shapes):
            raise ValueError(f"{len(names)} names vs {len(shapes)} shapes")
        self.names = list(names)
        self.shapes = [tuple(int(d) for d in s) for s in shapes]
        self.offsets: list[int] = []
        self.sizes: list[int] = []
        off = 0
        for s in self.shapes:
            n = math.prod(s)
            self.offsets.append(off)
            self.sizes.append(n)
            off += -(-n // self.ALIGN) * self.ALIGN if n else 0
        self.numel = off

    def __eq__(self, other) -> bool:
        return isinstance(other, FlatLayout) and self.shapes == other.shapes

    def views(self, buf: torch.Tensor) -> list[torch.Tensor]:
        return [buf[o : o + n].view(s) for o, n, s in zip(self.offsets, self.sizes, self.shapes)]

    def empty(self, device, zero: bool = False) -> torch.Tensor:
        if zero:
            return torch.zeros(self.numel, dtype=torch.float32, device=device)
        buf = torch.empty(self.numel, dtype=torch.float32, device=device)
        # keep the alignment padding deterministic (zero) without a full memset
        pad_ranges = self._padding()
        for lo, hi in pad_ranges:
            buf[lo:hi].zero_()
        return buf

    def _padding(self) -> list[tuple[int, int]]:
        out = []
        for i, (o, n) in enumerate(zip(self.offsets, self.sizes)):
            end = self.offsets[i + 1] if i + 1 < len(self.offsets) else self.numel
            if o + n < end:
                out.append((o + n, end))
        return out

    def pack(self, tensors: Sequence[torch.Tensor], device) -> torch.Tensor:
        """Copy a list of tensors (any device/dtype) into a new flat fp32 buffer."""
        buf = self.empty(device)
        for v, t in zip(self.views(buf), tensors):
            if tuple(t.shape) != v.shape:
                raise ValueError(f"shape {tuple(t.shape)} does not match layout {tuple(v.shape)}")
            v.copy_(t, non_blocking=True)
        return buf

    def locate(self, flat_index: int) -> str:
        for name, o, n in zip(self.names, self.offsets, self.sizes):
            if o <= flat_index < o + n:
                return name
        return "<padding>"

    def as_flat(self, tensors: Sequence[torch.Tensor]) -> torch.Tensor | None:
        """The flat buffer `tensors` are views of, if they are exactly this
        layout's views of one contiguous fp32 CUDA buffer; else None."""
        if len(tensors) != len(self.shapes) or not tensors:
            return None
        t0 = tensors[0]
        if t0.dtype != torch.float32 or not t0.is_cuda:
            return None
        st = t0.untyped_storage()
        base_ptr = t0.data_ptr() - self.offsets[0] * 4
        for t, o, s in zip(tensors, self.offsets, self.shapes):
            if (
                t.dtype != torch.float32
                or tuple(t.shape) != s
                or not t.is_contiguous()
                or t.untyped_storage().data_ptr() != st.data_ptr()
                or t.data_ptr() != base_ptr + 4 * o
            ):
                return None
        start = (base_ptr - st.data_ptr()) // 4
        if start < 0 or (start + self.numel) * 4 > st.nbytes():
            return None
        return torch.empty(0, dtype=torch.float32, device=t0.device).set_(
            st, start, (self.numel,), (1,)
        )


class FlatParams:
    """Live weights + gradient of one stage in flat device buffers."""

    def __init__(self, layout: FlatLayout, device, data: torch.Tensor | None = None):
        self.layout = layout
        self.device = torch.device(device)
        self.data = data if data is not None else layout.empty(self.device, zero=True)
        self.grad = layout.empty(self.device, zero=True)

    @classmethod
    def from_tensors(cls, names, tensors, device) -> "FlatParams":
        layout = FlatLayout(names, [tuple(t.shape) for t in tensors])
        return cls(layout, device, layout.pack(tensors, device))

    # per-parameter views are cached per buffer object (building ~2 views per
    # layer per event was ~30 % of the eager runners' host time)
    @property
    def params(self) -> list[torch.Tensor]:
        if getattr(self, "_pv_src", None) is not self.data:
            self._pv, self._pv_src = self.layout.views(self.data), self.data
        return self._pv

    @property
    def grads(self) -> list[torch.Tensor]:
        if getattr(self, "_gv_src", None) is not self.grad:
            self._gv, self._gv_src = self.layout.views(self.grad), self.grad
        return self._gv


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def _stream(device: torch.device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


# ---- the optimizer state ---------------------------------------------------------


class OptimizerState:
    """Per-stage optimizer state (optim.py:46-59) over a named list of params.

    step_count is the number of updates applied so far; the flat moment
    buffers are lazily zero-initialised on the first step (optim.py:91-92,
    103-105). `eager_checks=True` reproduces the reference's immediate
    NumericError on a non-finite step (one host sync per step); with False
    the flag accumulates on the device and `check_finite()` raises later.
    """

    def __init__(
        self,
        config: OptimizerConfig,
        names: list[str],
        *,
        device: torch.device | str | None = None,
        eager_checks: bool = True,
        launch: _lib.po_launch | None = None,
    ):
        self.config = config
        self.names = list(names)
        self.step_count = 0
        self.eager_checks = eager_checks
        self._device = torch.device(device) if device is not None else None
        self._layout: FlatLayout | None = None
        self._s1: torch.Tensor | None = None  # sgdm buf | adam exp_avg
        self._s2: torch.Tensor | None = None  # adam exp_avg_sq
        self._bad: torch.Tensor | None = None
        self._seg_flags: dict[int, torch.Tensor] = {}  # step_fused_ segment starts -> non-finite flags
        self._hp = config.hparams()
        self._launch = launch
        self._lib = _lib.load()
        # CUDA-graph mode: launches take their scalars from a CoefTape slot
        self.tape: "CoefTape | None" = None

    # -- state plumbing ---------------------------------------------------------

    @property
    def device(self) -> torch.device:
        if self._device is None:
            if not torch.cuda.is_available():
                raise _lib.LibraryMissing("PipeOptim kernels need a CUDA device (no CPU fallback)")
            self._device = torch.device("cuda", torch.cuda.current_device())
        return self._device

    def _bind(self, layout: FlatLayout) -> None:
        if self._layout is None:
            if len(layout.shapes) != len(self.names):
                raise ValueError(
                    f"{len(layout.shapes)} params vs {len(self.names)} names"
                )
            self._layout = FlatLayout(self.names, layout.shapes)
        elif self._layout != layout:
            raise ValueError("parameter shapes changed between optimizer calls")

    def _ensure_state(self) -> None:
        if self._s1 is None:
            self._s1 = self._layout.empty(self.device, zero=True)
            if self.config.kind != "sgdm":
                self._s2 = self._layout.empty(self.device, zero=True)
        if self._bad is None:
            self._bad = torch.full((1,), _INT64_MAX, dtype=torch.int64, device=self.device)

    def _state_views(self, buf):
        if buf is None or self._layout is None:
            return None
        return self._layout.views(buf)

    def _set_state(self, which: str, values) -> None:
        if values is None:
            setattr(self, which, None)
            return
        vals = [torch.as_tensor(v.a if hasattr(v, "a") else v) for v in values]
        self._bind(FlatLayout(self.names, [tuple(v.shape) for v in vals]))
        buf = getattr(self, which)
        if buf is None:
            buf = self._layout.empty(self.device, zero=True)
            setattr(self, which, buf)
        for dst, src in zip(self._layout.views(buf), vals):
            dst.copy_(src)

    @property
    def momentum_buf(self):
        return self._state_views(self._s1) if self.config.kind == "sgdm" else None

    @momentum_buf.setter
    def momentum_buf(self, values):
        self._set_state("_s1", values)

    @property
    def exp_avg(self):
        return self._state_views(self._s1) if self.config.kind != "sgdm" else None

    @exp_avg.setter
    def exp_avg(self, values):
        self._set_state("_s1", values)

    @property
    def exp_avg_sq(self):
        return self._state_views(self._s2) if self.config.kind != "sgdm" else None

    @exp_avg_sq.setter
    def exp_avg_sq(self, values):
        self._set_state("_s2", values)

    # -- non-finite reporting (optim.py:82-84) -----------------------------------

    def _after_step(self) -> None:
        if self.eager_checks:
            self.check_finite()

    def check_finite(self) -> None:
        """Raise NumericError naming the first parameter whose update went
        non-finite (flag set by the kernel); synchronises with the device."""
        if self._bad is None:
            return
        idx = int(self._bad.item())
        for lo, flag in self._seg_flags.items():  # segment launches of step_fused_
            j = int(flag.item())
            if j != _INT64_MAX:
                flag.fill_(_INT64_MAX)
                idx = min(idx, lo + j)
        if idx != _INT64_MAX:
            self._bad.fill_(_INT64_MAX)
            name = self._layout.locate(idx)
            raise NumericError(f"optimizer step produced non-finite values in {name}")

    # -- fast in-place paths on a FlatParams (the runtime's hot path) ------------

    def step_(self, flat: FlatParams, lr: float) -> None:
        """K2: one update in place on flat.data from flat.grad."""
        self._bind(flat.layout)
        self._ensure_state()
        if self.tape is not None:
            slot = self.tape.record(self, _lib.PO_COEF_STEP, lr, 0.0, 0)
            rc = self._lib.po_step_dc(
                ctypes.byref(self._hp), _ptr(flat.data), _ptr(flat.grad), _ptr(self._s1), _ptr(self._s2),
                flat.layout.numel, slot, _ptr(self._bad), self._launch_ref(), _stream(flat.data.device),
            )
            _lib.check(rc, "po_step_dc")
            self.step_count += 1
            return
        tok = AUDIT.before(self, "step", flat, None) if AUDIT is not None else None
        rc = self._lib.po_step(
            ctypes.byref(self._hp), _ptr(flat.data), _ptr(flat.grad), _ptr(self._s1),
            _ptr(self._s2), None, flat.layout.numel, float(lr), self.step_count,
            _ptr(self._bad), self._launch_ref(), _stream(flat.data.device),
        )
        _lib.check(rc, "po_step")
        if tok is not None:
            AUDIT.after(tok, lr, None, None)
        self._after_step()
        self.step_count += 1

    def predict_(self, flat: FlatParams, lr: float, steps_ahead: int, out: torch.Tensor) -> None:
        """K1: out = W - (lr*s) * dir(state), dir read at t = step_count."""
        if steps_ahead < 0:
            raise ValueError(f"steps_ahead must be >= 0, got {steps_ahead}")
        self._bind(flat.layout)
        if self.step_count > 0 or self.tape is not None:
            self._ensure_state()
        if self.tape is not None:
            slot = self.tape.record(self, _lib.PO_COEF_PREDICT, 0.0, lr, steps_ahead)
            rc = self._lib.po_predict_dc(
                ctypes.byref(self._hp), _ptr(flat.data), _ptr(self._s1), _ptr(self._s2), _ptr(out),
                flat.layout.numel, slot, self._launch_ref(), _stream(flat.data.device),
            )
            _lib.check(rc, "po_predict_dc")
            return
        tok = AUDIT.before(self, "predict", flat, out) if AUDIT is not None else None
        rc = self._lib.po_predict(
            ctypes.byref(self._hp), _ptr(flat.data), _ptr(self._s1), _ptr(self._s2), _ptr(out),
            flat.layout.numel, float(lr) * steps_ahead, self.step_count, self._launch_ref(),
            _stream(flat.data.device),
        )
        _lib.check(rc, "po_predict")
        if tok is not None:
            AUDIT.after(tok, None, lr, steps_ahead)

    def step_predict_(
        self, flat: FlatParams, lr: float, lr_pred: float, steps_ahead: int, out: torch.Tensor
    ) -> None:
        """K3: step_ then predict_ on the just-updated state, in one HBM pass."""
        if steps_ahead < 0:
            raise ValueError(f"steps_ahead must be >= 0, got {steps_ahead}")
        self._bind(flat.layout)
        self._ensure_state()
        if self.tape is not None:
            slot = self.tape.record(self, _lib.PO_COEF_STEP_PREDICT, lr, lr_pred, steps_ahead)
            rc = self._lib.po_step_predict_dc(
                ctypes.byref(self._hp), _ptr(flat.data), _ptr(flat.grad), _ptr(self._s1), _ptr(self._s2),
                _ptr(out), flat.layout.numel, slot, _ptr(self._bad), self._launch_ref(),
                _stream(flat.data.device),
            )
            _lib.check(rc, "po_step_predict_dc")
            self.step_count += 1
            return
        tok = AUDIT.before(self, "step_predict", flat, out) if AUDIT is not None else None
        rc = self._lib.po_step_predict(
            ctypes.byref(self._hp), _ptr(flat.data), _ptr(flat.grad), _ptr(self._s1),
            _ptr(self._s2), _ptr(out), flat.layout.numel, float(lr), float(lr_pred) * steps_ahead,
            self.step_count, _ptr(self._bad), self._launch_ref(), _stream(flat.data.device),
        )
        _lib.check(rc, "po_step_predict")
        if tok is not None:
            AUDIT.after(tok, lr, lr_pred, steps_ahead)
        self._after_step()
        self.step_count += 1

    def step_fused_(self, flat: FlatParams, lr: float, lr_pred: float, steps_ahead: int,
                    out: torch.Tensor | None, wgrad: list) -> None:
        """step_ (out None) or step_predict_ whose weight gradients for the
        params in `wgrad` — (param index, x, dpre) left by
        stage_backward(defer_wgrad=True) — are formed inside the update:
        po_wgrad_update computes x^T @ dpre on the tensor cores and applies
        K2/K3 in its epilogue; the other params (biases, unfused weights) go
        through K2/K3 from flat.grad, segment by segment. Same coefficients,
        same per-element rule, one step_count increment."""
        if steps_ahead < 0:
            raise ValueError(f"steps_ahead must be >= 0, got {steps_ahead}")
        self._bind(flat.layout)
        self._ensure_state()
        lay, dev = flat.layout, flat.data.device
        stream = _stream(dev)
        which = _lib.PO_COEF_STEP if out is None else _lib.PO_COEF_STEP_PREDICT
        coef = self.tape.record(self, which, lr, lr_pred, steps_ahead) if self.tape is not None else None
        c_pred = 0.0 if out is None else float(lr_pred) * steps_ahead
        hp = ctypes.byref(self._hp)
        fused = {}
        for idx, x, dpre in wgrad:
            fused[idx] = (x, dpre)
        for i, (o, n) in enumerate(zip(lay.offsets, lay.sizes)):
            if i not in fused:
                continue
            x, dpre = fused[i]
            rows, fin = x.shape
            fout = dpre.shape[1]
            rc = self._lib.po_wgrad_update(
                hp, _ptr(x), fin, _ptr(dpre), fout, rows, fin, fout, flat.data.data_ptr() + 4 * o,
                self._s1.data_ptr() + 4 * o, None if self._s2 is None else self._s2.data_ptr() + 4 * o,
                None if out is None else out.data_ptr() + 4 * o, None, float(lr), c_pred, self.step_count, coef,
                _ptr(self._bad), o, stream)
            _lib.check(rc, "po_wgrad_update")
        # the remaining params: maximal runs of consecutive non-fused params (padding included)
        i, k = 0, len(lay.offsets)
        while i < k:
            if i in fused:
                i += 1
                continue
            j = i
            while j + 1 < k and (j + 1) not in fused:
                j += 1
            lo = lay.offsets[i]
            hi = lay.offsets[j + 1] if j + 1 < k else lay.numel
            self._segment(flat, lo, hi - lo, lr, c_pred, out, coef, stream)
            i = j + 1
        if self.tape is None:
            self._after_step()
        self.step_count += 1

    def _segment(self, flat, lo, n, lr, c_pred, out, coef, stream) -> None:
        """K2/K3 on flat[lo : lo + n]. The kernels report a non-finite index
        relative to the launch, so each segment start has its own flag
        (`_seg_bad`), mapped back to the flat index by check_finite."""
        if n <= 0:
            return
        off = 4 * lo
        hp = ctypes.byref(self._hp)
        w, g, s1 = flat.data.data_ptr() + off, flat.grad.data_ptr() + off, self._s1.data_ptr() + off
        s2 = None if self._s2 is None else self._s2.data_ptr() + off
        bad = self._seg_bad(lo)
        if out is None:
            if coef is not None:
                rc = self._lib.po_step_dc(hp, w, g, s1, s2, n, coef, bad, self._launch_ref(), stream)
            else:
                rc = self._lib.po_step(hp, w, g, s1, s2, None, n, float(lr), self.step_count, bad,
                                       self._launch_ref(), stream)
        else:
            o = out.data_ptr() + off
            if coef is not None:
                rc = self._lib.po_step_predict_dc(hp, w, g, s1, s2, o, n, coef, bad, self._launch_ref(), stream)
            else:
                rc = self._lib.po_step_predict(hp, w, g, s1, s2, o, n, float(lr), c_pred, self.step_count, bad,
                                               self._launch_ref(), stream)
        _lib.check(rc, "po_step (segment)")

    def _seg_bad(self, lo: int) -> int:
        if lo == 0:
            return _ptr(self._bad)
        if lo not in self._seg_flags:
            self._seg_flags[lo] = torch.full((1,), _INT64_MAX, dtype=torch.int64, device=self.device)
        return self._seg_flags[lo].data_ptr()

    def _launch_ref(self):
        return ctypes.byref(self._launch) if self._launch is not None else None

    # -- reference-shaped list API ------------------------------------------------

    def _out(self, buf: torch.Tensor, host) -> list[torch.Tensor]:
        views = self._layout.views(buf)
        if host is None:
            return views
        outs = [torch.empty(v.shape, dtype=v.dtype, pin_memory=True) for v in views]
        for o, v in zip(outs, views):
            o.copy_(v, non_blocking=True)
        torch.cuda.current_stream(buf.device).synchronize()
        return outs

    def step(self, params, grads, lr: float):
        """Apply one update; returns (new params, applied directions) with
        new = old - lr*d (optim.py:63-87). Inputs are not mutated."""
        if len(params) != len(grads) or len(params) != len(self.names):
            raise ValueError(
                f"step: got {len(params)} params, {len(grads)} grads, "
                f"{len(self.names)} names"
            )
        params = [_as_tensor(p) for p in params]
        grads = [_as_tensor(g) for g in grads]
        layout = FlatLayout(self.names, [tuple(p.shape) for p in params])
        self._bind(layout)
        host = None if params[0].is_cuda else params[0].device
        if host is not None and all(not g.is_cuda for g in grads):
            return self._step_host(params, grads, lr)
        dev = params[0].device if params[0].is_cuda else self.device
        w = self._layout.pack(params, dev)  # a new buffer: inputs stay untouched
        g = self._layout.as_flat(grads) if host is None else None
        if g is None:
            g = self._layout.pack(grads, dev)
        self._ensure_state()
        dirs = self._layout.empty(dev)
        rc = self._lib.po_step(
            ctypes.byref(self._hp), _ptr(w), _ptr(g), _ptr(self._s1), _ptr(self._s2), _ptr(dirs),
            self._layout.numel, float(lr), self.step_count, _ptr(self._bad), self._launch_ref(),
            _stream(w.device),
        )
        _lib.check(rc, "po_step")
        self.check_finite()  # the list API always raises like the reference
        self.step_count += 1
        return self._out(w, host), self._out(dirs, host)

    def _streamer(self) -> "HostStreamer":
        if getattr(self, "_host_streamer", None) is None:
            self._host_streamer = _streamer_for(self.device, self._layout.numel)
        return self._host_streamer

    def _step_host(self, params, grads, lr):
        """step() on host tensors: W and G stream to the device in chunks and
        W' and the applied direction stream back (HostStreamer, three streams
        overlapped); the optimizer state never leaves the device. Outputs are
        new pinned host tensors (the inputs are not mutated)."""
        self._ensure_state()
        f32 = lambda t: t if t.dtype == torch.float32 else t.float()  # noqa: E731
        new_w = [torch.empty(p.shape, dtype=torch.float32, pin_memory=True) for p in params]
        dirs = [torch.empty(p.shape, dtype=torch.float32, pin_memory=True) for p in params]
        segs = [(o, f32(p).reshape(-1), f32(g).reshape(-1), w.reshape(-1), d.reshape(-1))
                for o, p, g, w, d in zip(self._layout.offsets, params, grads, new_w, dirs) if p.numel()]
        st = self._streamer()
        _, bad = st.run(self, "step_dir", segs, lr)
        torch.cuda.current_stream(self.device).synchronize()  # the outputs are host memory
        eager = self.eager_checks
        self.eager_checks = True  # the list API always raises like the reference
        try:
            st._raise_bad(self, bad, list(zip(self._layout.offsets, self._layout.sizes, self.names)))
        finally:
            self.eager_checks = eager
        self.step_count += 1
        return new_w, dirs

    def prediction_direction(self, params):
        """Direction the next update is expected to take, read from the
        buffers (optim.py:123-142): zeros before the first step, the momentum
        buffer for sgdm, (m/bc1)/(sqrt(v/bc2)+eps) at t = step_count for
        adam/adamw (no decoupled-decay term). Pure read."""
        params = [_as_tensor(p) for p in params]
        self._bind(FlatLayout(self.names, [tuple(p.shape) for p in params]))
        host = None if params[0].is_cuda else params[0].device
        dev = params[0].device if params[0].is_cuda else self.device
        if self.step_count > 0 and self._s1 is None:
            raise RuntimeError("prediction_direction: step_count > 0 but no optimizer state")
        out = self._layout.empty(dev)
        rc = self._lib.po_direction(
            ctypes.byref(self._hp), _ptr(self._s1), _ptr(self._s2), _ptr(out),
            self._layout.numel, self.step_count, self._launch_ref(), _stream(dev),
        )
        _lib.check(rc, "po_direction")
        return self._out(out, host)


class CoefTape:
    """Device-resident per-launch coefficients for CUDA-graph capture.

    While a graph is being captured, every K1/K2/K3 launch of an attached
    OptimizerState records (optimizer, kind, step count relative to the
    capture start, lr, lr*s) and gets a slot in a device po_coef array.
    Before each replay, `refresh()` recomputes every slot for the optimizer's
    CURRENT step count (host double arithmetic, `po_coef_fill`) and copies the
    array to the device on the replay stream, so replaying the graph
    continues training exactly as re-running the eager code would.
    """

    def __init__(self, device, capacity: int = 1 << 14):
        self.device = torch.device(device)
        self.capacity = capacity
        self.dev = torch.zeros(capacity * 4, dtype=torch.float32, device=self.device)
        # double-buffered pinned staging: a refresh never overwrites a buffer
        # whose H2D copy may still be pending
        self.host = [torch.zeros(capacity * 4, dtype=torch.float32).pin_memory() for _ in range(2)]
        self.copied = [None, None]
        self.flip = 0
        self.entries: list[tuple] = []
        self.base: dict[int, int] = {}
        self._lib = _lib.load()

    def begin(self, opts) -> None:
        """Start recording: remember each optimizer's step count at capture start."""
        self.entries.clear()
        self.base = {id(o): o.step_count for o in opts}
        for o in opts:
            o.tape = self

    def end(self, opts) -> None:
        for o in opts:
            o.tape = None

    def record(self, opt, which: int, lr, lr_pred, steps_ahead: int) -> int:
        """One launch's slot. `lr` / `lr_pred` may be `MbLr` values (a float
        that remembers the mini-batch it was computed for), in which case
        refresh() re-evaluates the learning-rate schedule for every replay."""
        i = len(self.entries)
        if i >= self.capacity:
            raise RuntimeError("CoefTape capacity exceeded")
        self.entries.append((opt, which, opt.step_count - self.base[id(opt)], lr, lr_pred, int(steps_ahead)))
        return self.dev.data_ptr() + 16 * i

    @staticmethod
    def _lr(value, lr_fn, mb_offset):
        mb = getattr(value, "mb", None)
        if lr_fn is None or mb is None:
            return float(value)
        return float(lr_fn(mb_offset + mb))

    def refresh(self, step_counts: dict[int, int], lr_fn=None, mb_offset: int = 0) -> None:
        """Fill every slot for the optimizers' step counts at replay start (and,
        with `lr_fn`, the schedule's learning rate at global mini-batch
        mb_offset + mb), in double on the host exactly as the eager calls."""
        k = self.flip
        self.flip ^= 1
        if self.copied[k] is not None:
            self.copied[k].synchronize()
        host = self.host[k]
        buf = (_lib.po_coef * self.capacity).from_address(host.data_ptr())
        for i, (opt, which, rel, lr, lr_pred, s) in enumerate(self.entries):
            a = self._lr(lr, lr_fn, mb_offset)
            c = self._lr(lr_pred, lr_fn, mb_offset) * s
            rc = self._lib.po_coef_fill(ctypes.byref(opt._hp), which, a, c, step_counts[id(opt)] + rel,
                                        ctypes.addressof(buf[i]))
            _lib.check(rc, "po_coef_fill")
        n = 4 * len(self.entries)
        if n:
            self.dev[:n].copy_(host[:n], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record()
            self.copied[k] = ev


class MbLr(float):
    """A learning rate that remembers the (run-local) mini-batch it is for, so a
    CUDA-graph replay can re-evaluate the schedule (CoefTape.refresh)."""

    def __new__(cls, value, mb):
        obj = super().__new__(cls, value)
        obj.mb = mb
        return obj


class HostStreamer:
    """Host-buffer path for one flat stage: pinned host W and G stream to the
    device in chunks, K3 runs on each chunk against the device-resident
    optimizer state, and the updated W and the prediction W_hat stream back —
    H2D, compute and D2H on three streams with `slots`-deep buffering so the
    PCIe transfers in both directions overlap each other and the kernel.
    This is what a caller that keeps parameters on the host sees end to end.
    """

    def __init__(self, device, chunk_elems: int = 1 << 24, slots: int = 4):
        self.device = torch.device(device)
        self.chunk = int(chunk_elems)
        self.slots = int(slots)
        mk = lambda: [torch.empty(self.chunk, dtype=torch.float32, device=self.device) for _ in range(self.slots)]  # noqa: E731
        self.dw, self.dg, self.dwh = mk(), mk(), mk()
        self.s_in = torch.cuda.Stream(self.device)
        self.s_comp = torch.cuda.Stream(self.device)
        self.s_out = torch.cuda.Stream(self.device)
        self.ev_in = [torch.cuda.Event() for _ in range(self.slots)]
        self.ev_comp = [torch.cuda.Event() for _ in range(self.slots)]
        self.ev_free = [None] * self.slots

    def step_predict(self, opt: "OptimizerState", w_host: torch.Tensor, g_host: torch.Tensor, lr: float,
                     lr_pred: float, steps_ahead: int, w_out: torch.Tensor, w_hat_out: torch.Tensor) -> int:
        """K3 over host buffers (1-D fp32, pinned). Returns the kernel launch count."""
        n = w_host.numel()
        if steps_ahead < 0:
            raise ValueError(f"steps_ahead must be >= 0, got {steps_ahead}")
        opt._bind(FlatLayout(opt.names, [(n,)]))
        opt._ensure_state()
        launches, bad = self.run(opt, "step_predict", [(0, w_host, g_host, w_out, w_hat_out)], lr,
                                 float(lr_pred) * steps_ahead)
        self._raise_bad(opt, bad, [(0, n, opt.names[0])])
        opt.step_count += 1
        return launches

    def run(self, opt: "OptimizerState | None", mode: str, segs, lr: float = 0.0, c_pred: float = 0.0):
        """Stream host segments through the device in chunks: H2D on one
        stream, the kernel per chunk on another, D2H on a third, `slots`-deep
        buffers, so both PCIe directions and the kernel overlap. Each segment
        is (state offset, a_host, b_host, out1_host, out2_host), all 1-D fp32:

          "step_predict"  a = W, b = G  -> out1 = W', out2 = W_hat   (K3)
          "step_dir"      a = W, b = G  -> out1 = W', out2 = dir     (K2 + dir)
          "axpy"          a = W, b = d  -> out1 = W - c_pred * d     (predict_weights)

        The optimizer state (K2/K3) stays on the device at the segment's
        offset. Returns (launches, per-chunk non-finite flags on the device)."""
        chunks = []
        for off, a, b, o1, o2 in segs:
            for lo in range(0, a.numel(), self.chunk):
                chunks.append((off, a, b, o1, o2, lo, min(self.chunk, a.numel() - lo)))
        bad = torch.full((max(1, len(chunks)),), _INT64_MAX, dtype=torch.int64, device=self.device)
        cur = torch.cuda.current_stream(self.device)
        for st in (self.s_in, self.s_comp, self.s_out):
            st.wait_stream(cur)
        lib = _lib.load()
        hp = ctypes.byref(opt._hp) if opt is not None else None
        la = opt._launch_ref() if opt is not None else None
        for i, (off, a, b, o1, o2, lo, m) in enumerate(chunks):
            k = i % self.slots
            with torch.cuda.stream(self.s_in):
                if self.ev_free[k] is not None:
                    self.s_in.wait_event(self.ev_free[k])
                self.dw[k][:m].copy_(a[lo : lo + m], non_blocking=True)
                self.dg[k][:m].copy_(b[lo : lo + m], non_blocking=True)
                self.ev_in[k].record(self.s_in)
            self.s_comp.wait_event(self.ev_in[k])
            sc = self.s_comp.cuda_stream
            if mode == "axpy":
                rc = lib.po_axpy_predict(_ptr(self.dw[k]), _ptr(self.dg[k]), _ptr(self.dwh[k]), m, float(c_pred),
                                         None, sc)
            else:
                s1 = opt._s1[off + lo:].data_ptr()
                s2 = opt._s2[off + lo:].data_ptr() if opt._s2 is not None else None
                if mode == "step_predict":
                    rc = lib.po_step_predict(hp, _ptr(self.dw[k]), _ptr(self.dg[k]), s1, s2, _ptr(self.dwh[k]), m,
                                             float(lr), float(c_pred), opt.step_count, bad[i:].data_ptr(), la, sc)
                elif mode == "step_dir":
                    rc = lib.po_step(hp, _ptr(self.dw[k]), _ptr(self.dg[k]), s1, s2, _ptr(self.dwh[k]), m,
                                     float(lr), opt.step_count, bad[i:].data_ptr(), la, sc)
                else:
                    raise ValueError(f"unknown streaming mode {mode!r}")
            _lib.check(rc, f"HostStreamer.run({mode})")
            self.ev_comp[k].record(self.s_comp)
            with torch.cuda.stream(self.s_out):
                self.s_out.wait_event(self.ev_comp[k])
                if mode == "axpy":
                    o1[lo : lo + m].copy_(self.dwh[k][:m], non_blocking=True)
                else:
                    o1[lo : lo + m].copy_(self.dw[k][:m], non_blocking=True)
                    o2[lo : lo + m].copy_(self.dwh[k][:m], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(self.s_out)
                self.ev_free[k] = ev
        cur.wait_stream(self.s_out)
        # (offset, start, length) only: holding the chunks' host tensors here
        # would keep the caller's dropped outputs out of torch's pinned-host
        # cache until the next call, which would then pin fresh memory
        self._chunks = [(off, lo, m) for off, _a, _b, _o1, _o2, lo, m in chunks]
        return len(chunks), bad

    def _raise_bad(self, opt, bad, where) -> None:
        """eager_checks: sync and raise NumericError for the first non-finite
        chunk, naming the parameter (`where`: (state offset, numel, name))."""
        if not opt.eager_checks:
            return
        torch.cuda.current_stream(self.device).synchronize()
        for (off, lo, m), v in zip(self._chunks, bad.cpu().tolist()):
            if v != _INT64_MAX:
                name = next((nm for o, n, nm in where if o <= off + lo + v < o + n), opt.names[0])
                raise NumericError(f"optimizer step produced non-finite values in {name}")

    def step_predict_resident(self, opt: "OptimizerState", w_dev: torch.Tensor, g_host: torch.Tensor, lr: float,
                              lr_pred: float, steps_ahead: int, w_hat_dev: torch.Tensor) -> int:
        """K3 with the weights and state device-resident and only the gradient
        on the host (pinned): G streams in chunk by chunk, each chunk's K3
        starts as soon as it lands; W' and W_hat stay on the device. Returns
        the launch count; the non-finite flag is the only device->host read."""
        n = g_host.numel()
        if steps_ahead < 0:
            raise ValueError(f"steps_ahead must be >= 0, got {steps_ahead}")
        opt._bind(FlatLayout(opt.names, [(n,)]))
        opt._ensure_state()
        n_chunks = -(-n // self.chunk)
        cur = torch.cuda.current_stream(self.device)
        self.s_in.wait_stream(cur)
        self.s_comp.wait_stream(cur)
        hp = ctypes.byref(opt._hp)
        c_pred = float(lr_pred) * steps_ahead
        for i in range(n_chunks):
            k = i % self.slots
            lo = i * self.chunk
            m = min(self.chunk, n - lo)
            with torch.cuda.stream(self.s_in):
                if self.ev_free[k] is not None:
                    self.s_in.wait_event(self.ev_free[k])
                self.dg[k][:m].copy_(g_host[lo : lo + m], non_blocking=True)
                self.ev_in[k].record(self.s_in)
            self.s_comp.wait_event(self.ev_in[k])
            rc = opt._lib.po_step_predict(
                hp, w_dev[lo:].data_ptr(), _ptr(self.dg[k]), opt._s1[lo:].data_ptr(),
                None if opt._s2 is None else opt._s2[lo:].data_ptr(), w_hat_dev[lo:].data_ptr(), m, float(lr),
                c_pred, opt.step_count, opt._bad.data_ptr(), opt._launch_ref(), self.s_comp.cuda_stream,
            )
            _lib.check(rc, "po_step_predict")
            ev = torch.cuda.Event()
            ev.record(self.s_comp)
            self.ev_free[k] = ev
        cur.wait_stream(self.s_comp)
        opt._after_step()  # eager_checks: raise NumericError now, like step_predict
        opt.step_count += 1
        return n_chunks


def _as_tensor(x) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        return x
    a = getattr(x, "a", x)  # a reference Matrix carries its array in .a
    return torch.as_tensor(a)


_STREAMERS: dict = {}


def _streamer_for(device, numel: int) -> HostStreamer:
    """A cached HostStreamer whose chunk fits `numel` (<= 16 M elements):
    small host calls do not pin down 3 x 4 x 64 MB of device buffers."""
    device = torch.device(device)
    chunk = min(1 << 24, max(1 << 12, 1 << max(0, int(numel) - 1).bit_length()))
    key = (device.index, chunk)
    if key not in _STREAMERS:
        _STREAMERS[key] = HostStreamer(device, chunk_elems=chunk)
    return _STREAMERS[key]


def predict_weights(params, lr: float, steps_ahead: int, directions) -> list[torch.Tensor]:
    """Extrapolate parameters steps_ahead updates into the future: each w
    becomes w - lr * steps_ahead * d (optim.py:145-155, Eq. (5)). Inputs are
    not mutated."""
    if steps_ahead < 0:
        raise ValueError(f"steps_ahead must be >= 0, got {steps_ahead}")
    if len(params) != len(directions):
        raise ValueError(
            f"predict_weights: {len(params)} params vs {len(directions)} directions"
        )
    if not params:
        return []
    params = [_as_tensor(p) for p in params]
    directions = [_as_tensor(d) for d in directions]
    names = [f"p{i}" for i in range(len(params))]
    layout = FlatLayout(names, [tuple(p.shape) for p in params])
    host = None if params[0].is_cuda else params[0].device
    if host is not None and all(not d.is_cuda for d in directions):
        # host tensors: W and d stream through the device chunk by chunk
        dev = torch.device("cuda", torch.cuda.current_device())
        st = _streamer_for(dev, layout.numel)
        f32 = lambda t: t if t.dtype == torch.float32 else t.float()  # noqa: E731
        outs = [torch.empty(p.shape, dtype=torch.float32, pin_memory=True) for p in params]
        st.run(None, "axpy", [(0, f32(p).reshape(-1), f32(d).reshape(-1), o.reshape(-1), None)
                              for p, d, o in zip(params, directions, outs) if p.numel()],
               c_pred=float(lr) * steps_ahead)
        torch.cuda.current_stream(dev).synchronize()
        return outs
    dev = params[0].device if params[0].is_cuda else torch.device("cuda", torch.cuda.current_device())
    w = layout.as_flat(params) if host is None else None
    if w is None:
        w = layout.pack(params, dev)
    d = layout.as_flat(directions) if host is None else None
    if d is None:
        d = layout.pack(directions, dev)
    out = layout.empty(dev)
    lib = _lib.load()
    rc = lib.po_axpy_predict(
        _ptr(w), _ptr(d), _ptr(out), layout.numel, float(lr) * steps_ahead, None, _stream(dev)
    )
    _lib.check(rc, "po_axpy_predict")
    views = layout.views(out)
    return views if host is None else [v.to(host) for v in views]


def version_difference(depth: int, rank: int) -> int:
    """Eq. (4): updates a stage applies between a mini-batch's forward and its
    backward in 1F1B steady state, depth - rank - 1 (optim.py:158-167)."""
    if depth < 1:
        raise ValueError(f"depth must be >= 1, got {depth}")
    if not 0 <= rank < depth:
        raise ValueError(f"rank must be in [0, {depth}), got {rank}")
    out = ctypes.c_int64(0)
    _lib.check(_lib.load().po_version_difference(depth, rank, ctypes.byref(out)), "version_difference")
    return int(out.value)
