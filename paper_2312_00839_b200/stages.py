"""Dense-MLP pipeline stages on the device, with the reference's weight-view
semantics.

Mirrors pkg/src/pipesim/stages.py: `LayerSpec`, `build_layers`,
`partition_layers` (contiguous, earlier stages take the extra layer),
`StageModel` (params [w0, b0, w1, b1, ...], w shaped (in, out) used as
x @ w + b, version starting at 1), the per-(mb, micro) `ActivationStash`, and
`stage_forward` / `stage_backward`.

The semantics that matter for parity: the forward runs on
whatever weights view the policy hands it (live or predicted W_hat) and
stashes layer inputs and pre-activations; the backward computes
dW = x^T dpre and db = colsum(dpre) from the stash, and the input gradient
with the weights view given at BACKWARD time (live weights under PipeOptim,
runtime.py:260-261, stages.py:200-208).

B200 layout: a stage's parameters live in one flat fp32 buffer (FlatParams)
so the optimizer/predictor kernels stream the whole stage in one launch; the
backward writes parameter gradients straight into the flat gradient buffer's
views (no separate accumulation pass for one micro-batch per update).
"""

from __future__ import annotations

import contextlib
from dataclasses import dataclass
from typing import Callable

import torch

from .errors import DimensionError, NumericError, StashError
from .optim import FlatParams

ACTIVATIONS = ("tanh", "relu", "linear")


@dataclass(frozen=True)
class LayerSpec:
    index: int
    in_dim: int
    out_dim: int
    activation: str

    def __post_init__(self):
        if self.activation not in ACTIVATIONS:
            raise ValueError(f"unknown activation kind: {self.activation!r}")
        if self.in_dim < 1 or self.out_dim < 1:
            raise ValueError(
                f"layer {self.index}: dims must be positive, got {self.in_dim}x{self.out_dim}"
            )


def build_layers(layer_dims: list[int], activations: list[str]) -> list[LayerSpec]:
    """MLP layer specs from a dim chain (stages.py:48-60)."""
    if len(layer_dims) < 2:
        raise ValueError("layer_dims needs at least an input and an output dim")
    if len(activations) != len(layer_dims) - 1:
        raise ValueError(
            f"expected {len(layer_dims) - 1} activations for {len(layer_dims)} dims, "
            f"got {len(activations)}"
        )
    return [LayerSpec(i, a, b, act) for i, (a, b, act) in enumerate(zip(layer_dims, layer_dims[1:], activations))]


def partition_layers(layers: list[LayerSpec], depth: int) -> list[list[LayerSpec]]:
    """Contiguous split, sizes differ by <= 1, earlier stages take the extra
    layer (stages.py:63-80)."""
    if depth < 1:
        raise ValueError(f"depth must be >= 1, got {depth}")
    if depth > len(layers):
        raise ValueError(f"cannot split {len(layers)} layers across {depth} stages")
    q, r = divmod(len(layers), depth)
    bounds = [0]
    for k in range(depth):
        bounds.append(bounds[-1] + q + (1 if k < r else 0))
    return [layers[bounds[k] : bounds[k + 1]] for k in range(depth)]


# An init provider maps a LayerSpec to (w (in, out), b (1, out)) — e.g. the
# reference's per-layer Philox substreams for parity runs (stages.py:83-91),
# or `torch_init` for synthetic throughput runs.
InitFn = Callable[[LayerSpec], tuple]


def torch_init(seed: int = 0, device="cpu") -> InitFn:
    """N(0, 1) * in_dim^-1/2 weights, zero bias, one generator per layer so the
    values do not depend on the partition (same distribution as stages.py:83-91,
    different RNG)."""

    def init(spec: LayerSpec):
        g = torch.Generator(device=device)
        g.manual_seed(seed * 1_000_003 + spec.index)
        w = torch.randn(spec.in_dim, spec.out_dim, generator=g, device=device) * spec.in_dim ** -0.5
        return w, torch.zeros(1, spec.out_dim, device=device)

    return init


@dataclass
class StashEntry:
    version: int
    layer_inputs: list
    pre_acts: list


class ActivationStash:
    """Forward context per (mb, micro) until the matching backward (stages.py:101-120)."""

    def __init__(self):
        self._entries: dict[tuple[int, int], StashEntry] = {}
        self.peak = 0

    def put(self, key, entry: StashEntry) -> None:
        if key in self._entries:
            raise StashError(f"stash already holds an entry for {key}")
        self._entries[key] = entry
        self.peak = max(self.peak, len(self._entries))

    def pop(self, key) -> StashEntry:
        try:
            return self._entries.pop(key)
        except KeyError:
            raise StashError(f"no stash entry for {key}") from None

    def __len__(self) -> int:
        return len(self._entries)


class StageModel:
    """One pipeline stage: its layers, live parameters in a flat device buffer,
    a version counter (starts at 1, +1 per update) and the activation stash."""

    def __init__(self, rank: int, layers: list[LayerSpec], init: InitFn, device=None):
        self.rank = rank
        self.layers = list(layers)
        self.device = torch.device(device) if device is not None else torch.device("cuda")
        names, tensors = [], []
        for spec in self.layers:
            w, b = init(spec)
            w = torch.as_tensor(getattr(w, "a", w))
            b = torch.as_tensor(getattr(b, "a", b))
            if tuple(w.shape) != (spec.in_dim, spec.out_dim) or tuple(b.shape) != (1, spec.out_dim):
                raise DimensionError(
                    f"layer {spec.index}: init shapes {tuple(w.shape)}, {tuple(b.shape)} "
                    f"vs ({spec.in_dim}, {spec.out_dim}), (1, {spec.out_dim})"
                )
            names += [f"layer{spec.index}.w", f"layer{spec.index}.b"]
            tensors += [w, b]
        self.param_names = names
        self.flat = FlatParams.from_tensors(names, tensors, self.device)
        self.version = 1
        self.stash = ActivationStash()

    @property
    def params(self) -> list[torch.Tensor]:
        return self.flat.params

    @params.setter
    def params(self, values) -> None:
        for dst, src in zip(self.flat.params, values):
            if dst.data_ptr() != src.data_ptr():
                dst.copy_(src)

    @property
    def in_dim(self) -> int:
        return self.layers[0].in_dim

    @property
    def out_dim(self) -> int:
        return self.layers[-1].out_dim

    @property
    def numel(self) -> int:
        return self.flat.layout.numel

    @property
    def in_shape(self) -> tuple:
        return (self.in_dim,)

    @property
    def out_shape(self) -> tuple:
        return (self.out_dim,)

    def set_grad_buffer(self, buf: torch.Tensor) -> None:
        """Point the stage's flat gradient at `buf` (same layout), e.g. the
        current parity of a fused-DP double buffer."""
        self.flat.grad = buf

    def set_weight_buffer(self, buf: torch.Tensor) -> None:
        """Move the live weights into `buf` (same layout), e.g. a peer-mapped
        buffer the sharded DP update writes into."""
        buf.copy_(self.flat.data)
        self.flat.data = buf

    def run_forward(self, weights, key, x, version, check_finite=True, finite_flags=None, flag_index=0):
        return stage_forward(self, weights, key, x, version, check_finite, finite_flags, flag_index)

    def run_forward_loss(self, weights, key, x, version, target, loss_kind, check_finite=True, finite_flags=None,
                         flag_index=0):
        """The last stage's forward followed by the loss (runtime.py:415-426):
        (out, loss, dL/dout). A narrow output layer runs forward, loss and
        gradient in one launch (po_head_fwd_loss, bit-identical to
        run_forward + loss_and_grad); otherwise the two calls."""
        req = {"y": target, "kind": loss_kind} if FUSED_HEAD_LOSS else None
        out = stage_forward(self, weights, key, x, version, check_finite, finite_flags, flag_index, loss_req=req)
        if req is not None and "loss" in req:
            return out, req["loss"], req["grad"]
        loss, grad = loss_and_grad(out, target, loss_kind)
        return out, loss, grad

    def run_backward(self, weights, key, grad_out, accumulate=False, need_input_grad=True, defer_wgrad=False):
        return stage_backward(self, weights, key, grad_out, accumulate, need_input_grad, defer_wgrad)

    def take_deferred_wgrad(self) -> list:
        """The (param index, x, dpre) the last backward left for the update."""
        d = getattr(self, "deferred_wgrad", None) or []
        self.deferred_wgrad = []
        return d


def build_stages(layers: list[LayerSpec], depth: int, init: InitFn, device=None) -> list[StageModel]:
    return [StageModel(k, group, init, device) for k, group in enumerate(partition_layers(layers, depth))]


def _activate(pre: torch.Tensor, kind: str) -> torch.Tensor:
    if kind == "tanh":
        return torch.tanh(pre)
    if kind == "relu":
        return torch.relu(pre)
    return pre


def _activation_grad_mul(g: torch.Tensor, pre: torch.Tensor, kind: str) -> torch.Tensor:
    """g * act'(pre) (linalg.py:185-194 then hadamard)."""
    if kind == "tanh":
        t = torch.tanh(pre)
        return g * (1.0 - t * t)
    if kind == "relu":
        return g * (pre > 0.0)  # one multiply with the mask promoted in-kernel
    return g


_ACT_CODE = {"linear": 0, "relu": 1, "tanh": 2}


def _splitk(rows: int, k: int, n: int) -> int:
    """Split count for a GEMM of `rows` x k @ k x n on the device: the 1F1B
    stages multiply a batch of ~128 rows by wide weights, a long-K, few-tile
    shape cuBLAS runs on a handful of CTAs (scripts/gemm_splitk.py: 3072x1024
    59 us as one GEMM, 19 us as 8 batched K-slices). Split K into S power-of-
    two slices of >= 256 (>= 32 for narrow outputs) while S <= 8 (32)."""
    if rows > 512 or k < 512:
        return 1
    cap, floor = (32, 32) if n < 64 else (8, 256)
    s = 1
    while s * 2 <= cap and k % (s * 2) == 0 and k // (s * 2) >= floor:
        s *= 2
    return s


# fp32 stage GEMMs on the tensor cores (csrc/pipeoptim_gemm.cu: tcgen05 UMMA,
# each fp32 operand split into three bf16 pieces — fp32-level accuracy) when
# TF32 is off; set False to use cuBLAS's SIMT SGEMM instead.
TC_FP32 = True


_TC_BUILT: bool | None = None


def _tc_built() -> bool:
    """po_gemm_f32x3 was compiled (the library found CUTLASS at build time)."""
    global _TC_BUILT
    if _TC_BUILT is None:
        from . import _lib

        _TC_BUILT = bool(_lib.load().po_gemm_f32x3_available())
    return _TC_BUILT


def _tc_ok(*tensors) -> bool:
    return (TC_FP32 and not torch.backends.cuda.matmul.allow_tf32
            and all(t.is_cuda and t.dtype == torch.float32 and t.data_ptr() % 16 == 0 for t in tensors)
            and _tc_built())


# Most K slices of a tensor-core GEMM's split-K (forward and input gradient):
# 8 is the latency-optimal count for a stage alone on its GPU; runners whose
# stages share one GPU lower it (runtime.SHARED_GPU_SPLIT_CAP) through
# gemm_split_cap(). The count only regroups fp32 partial sums.
TC_SPLIT_CAP = 8
_tc_split_cap = TC_SPLIT_CAP


@contextlib.contextmanager
def gemm_split_cap(cap: int):
    """Cap the tensor-core GEMMs' K slices at `cap` (a power of two >= 1)
    for the duration (decided when a forward / backward is issued or
    captured into a CUDA graph)."""
    global _tc_split_cap
    cap = int(cap)
    if cap < 1 or cap & (cap - 1):
        raise ValueError(f"gemm split cap must be a power of two >= 1, got {cap}")
    old, _tc_split_cap = _tc_split_cap, cap
    try:
        yield
    finally:
        _tc_split_cap = old


@contextlib.contextmanager
def gemm_tile(tile_n: int | None):
    """Tile width (64 or 128 output columns) of the tensor-core GEMMs for the
    duration (po_set_gemm_tile; None leaves the current one). 64: most CTAs,
    lowest latency (a stage alone on its GPU); 128: half the CTAs, less SM
    time (stages sharing one GPU)."""
    if tile_n is None:
        yield
        return
    from . import _lib

    lib = _lib.load()
    old = lib.po_get_gemm_tile()
    _lib.check(lib.po_set_gemm_tile(int(tile_n)), "po_set_gemm_tile")
    try:
        yield
    finally:
        lib.po_set_gemm_tile(old)


def _splitk_tc(rows: int, k: int) -> int:
    """K slices for the tensor-core GEMM of a small-M long-K shape: <= 8
    slices of >= 128 (scripts/gemm_f32x3_check.py: 3072x1024 forward 14 us at
    8 slices vs 19 us for the best SIMT split), capped by gemm_split_cap."""
    if rows > 512 or k < 256:
        return 1
    s = 1
    while s < _tc_split_cap and k % (s * 2) == 0 and k // (s * 2) >= 128:
        s *= 2
    return s


def _gemm_tc(a, a_col: bool, lda: int, sa: int, b, b_col: bool, ldb: int, sb: int, m: int, n: int, k: int,
             batch: int, out: torch.Tensor) -> torch.Tensor:
    from . import _lib

    rc = _lib.load().po_gemm_f32x3(int(a_col), int(b_col), a.data_ptr(), lda, sa, b.data_ptr(), ldb, sb,
                                   out.data_ptr(), m, n, k, batch, None, 0,
                                   torch.cuda.current_stream(out.device).cuda_stream)
    _lib.check(rc, "po_gemm_f32x3")
    return out


def _splitk_reduce(part: torch.Tensor, bias, act: str, pre_out=None, flags=None, flag_index: int = 0):
    """act(sum_s part[s] + bias) in one launch (po_splitk_bias_act); with
    `flags`, flags[flag_index] is cleared if any output is non-finite."""
    from . import _lib

    splits, rows, cols = part.shape
    out = torch.empty((rows, cols), dtype=torch.float32, device=part.device)
    rc = _lib.load().po_splitk_bias_act(part.data_ptr(), splits, rows, cols,
                                        None if bias is None else bias.data_ptr(), _ACT_CODE[act], out.data_ptr(),
                                        None if pre_out is None else pre_out.data_ptr(),
                                        None if flags is None else flags.data_ptr(), flag_index,
                                        torch.cuda.current_stream(part.device).cuda_stream)
    _lib.check(rc, "po_splitk_bias_act")
    return out


# Narrow linear layers (out <= 32: config 1's classifier) on po_head_fwd /
# po_head_bwd — one launch each way — instead of the library GEMMs (A/B switch)
FUSED_HEAD = True
# ... and, on the last stage (run_forward_loss), its forward + loss + dL/dout
# in ONE launch (po_head_fwd_loss) instead of po_head_fwd + po_loss_grad
FUSED_HEAD_LOSS = True


def _head_ok(h: torch.Tensor, w: torch.Tensor, act: str) -> bool:
    from . import _lib

    return (FUSED_HEAD and act == "linear" and h.is_cuda and h.dtype == torch.float32 and w.is_contiguous()
            and _lib.load().po_head_supported(h.shape[0], h.shape[1], w.shape[1]) == 1)


def _head_loss_ok(req, rows: int, n: int, device) -> bool:
    """The fused head forward + loss applies: a valid loss kind and an fp32
    contiguous target of the output's shape on the same device."""
    if req is None or req["kind"] not in LOSS_KINDS:
        return False
    y = req["y"]
    return (isinstance(y, torch.Tensor) and y.dtype == torch.float32 and y.is_contiguous()
            and y.device == device and tuple(y.shape) == (rows, n))


def _affine(h: torch.Tensor, w: torch.Tensor, b: torch.Tensor, act: str, flags=None, flag_index: int = 0,
            loss_req=None):
    """Device forward of one layer: (pre, h_out, checked) with the stash's
    convention — relu layers stash relu(pre) (its sign pattern is pre's),
    others pre. checked: the finiteness flag was already written (split-K
    epilogue / head kernel). loss_req ({"y", "kind"}, last layer only): a
    narrow output layer also computes the loss and dL/dout in its launch
    (po_head_fwd_loss) and stores them under "loss" / "grad"."""
    rows, k = h.shape
    n = w.shape[1]
    h = h if h.is_contiguous() else h.contiguous()
    if _head_ok(h, w, act):  # narrow linear layer: one launch (po_head_fwd)
        from . import _lib

        out = torch.empty((rows, n), dtype=torch.float32, device=h.device)
        bias = b.reshape(-1)
        stream = torch.cuda.current_stream(h.device).cuda_stream
        fl = None if flags is None else flags.data_ptr()
        if _head_loss_ok(loss_req, rows, n, h.device):
            key = (h.device, rows, stream)  # loss_and_grad's scratch (per device, rows, stream)
            if key not in _LOSS_SCRATCH:
                _LOSS_SCRATCH[key] = torch.zeros(rows + 1, dtype=torch.float32, device=h.device)
            grad = torch.empty_like(out)
            loss = torch.empty((), dtype=torch.float32, device=h.device)
            code = _lib.PO_LOSS_MSE if loss_req["kind"] == "mse" else _lib.PO_LOSS_SOFTMAX_XENT
            rc = _lib.load().po_head_fwd_loss(h.data_ptr(), rows, k, w.data_ptr(), bias.data_ptr(), n,
                                              loss_req["y"].data_ptr(), code, out.data_ptr(), grad.data_ptr(),
                                              loss.data_ptr(), _LOSS_SCRATCH[key].data_ptr(), fl, flag_index, stream)
            _lib.check(rc, "po_head_fwd_loss")
            loss_req["loss"], loss_req["grad"] = loss, grad
            return out, out, flags is not None
        rc = _lib.load().po_head_fwd(h.data_ptr(), rows, k, w.data_ptr(), bias.data_ptr(), n, out.data_ptr(), fl,
                                     flag_index, stream)
        _lib.check(rc, "po_head_fwd")
        return out, out, flags is not None
    tc = n % 4 == 0 and k % 4 == 0 and _tc_ok(h, w)
    s = _splitk_tc(rows, k) if tc else _splitk(rows, k, n)
    if tc:  # tensor-core fp32 GEMM, batch = K slice, into the fused epilogue
        part = _gemm_tc(h, False, k, k // s, w, False, n, (k // s) * n, rows, n, k // s, s,
                        torch.empty((s, rows, n), dtype=torch.float32, device=h.device))
    elif s > 1:
        part = torch.bmm(h.view(rows, s, k // s).transpose(0, 1), w.view(s, k // s, n))
    if tc or s > 1:
        bias = b.view(-1)
        if act == "tanh":
            pre = torch.empty((rows, n), dtype=torch.float32, device=h.device)
            return pre, _splitk_reduce(part, bias, act, pre_out=pre, flags=flags, flag_index=flag_index), \
                flags is not None
        out = _splitk_reduce(part, bias, act, flags=flags, flag_index=flag_index)
        return out, out, flags is not None
    if act == "relu":
        out = torch._addmm_activation(b.view(-1), h, w)
        return out, out, False
    pre = torch.addmm(b.view(-1), h, w)
    return pre, _activate(pre, act), False


def _input_grad_parts(dpre: torch.Tensor, w: torch.Tensor) -> torch.Tensor:
    """dpre @ w^T on the device as [splits, rows, in] partial products,
    split-K over the layer's output width (splits = 1: the product itself)."""
    rows, n = dpre.shape
    k = w.shape[0]
    dpre = dpre if dpre.is_contiguous() else dpre.contiguous()
    if n % 4 == 0 and k % 4 == 0 and _tc_ok(dpre, w):  # W^T read K-major straight from the flat buffer
        s = _splitk_tc(rows, n)
        return _gemm_tc(dpre, False, n, n // s, w, True, n, n // s, rows, k, n // s, s,
                        torch.empty((s, rows, k), dtype=torch.float32, device=dpre.device))
    s = _splitk(rows, n, k)
    if s > 1:
        return torch.bmm(dpre.view(rows, s, n // s).transpose(0, 1), w.view(k, s, n // s).permute(1, 2, 0))
    return torch.mm(dpre, w.t()).unsqueeze(0)


def _weight_grad(x: torch.Tensor, dpre: torch.Tensor, gw: torch.Tensor, accumulate: bool) -> None:
    """gw (=|+=) x^T @ dpre: the tensor-core fp32 GEMM reads x^T M-major
    straight from the stashed activation and writes the flat-gradient view."""
    rows, k_in = x.shape
    n = dpre.shape[1]
    if (not accumulate and n % 4 == 0 and k_in % 4 == 0 and gw.is_contiguous() and x.is_contiguous()
            and dpre.is_contiguous() and _tc_ok(x, dpre, gw)):
        _gemm_tc(x, True, k_in, 0, dpre, False, n, 0, k_in, n, rows, 1, gw)
    elif accumulate:
        gw.addmm_(x.t(), dpre)
    else:
        torch.mm(x.t(), dpre, out=gw)


def _input_grad(dpre: torch.Tensor, w: torch.Tensor) -> torch.Tensor:
    """dpre @ w^T on the device (split-K partials reduced in one launch)."""
    part = _input_grad_parts(dpre, w)
    return part[0] if part.shape[0] == 1 else _splitk_reduce(part, None, "linear")


_SIDE: dict = {}


def _side_stream(device) -> "torch.cuda.Stream":
    """One auxiliary stream per device per CURRENT stream (cached), for work
    that only reads a tensor the main stream also reads."""
    key = (device, torch.cuda.current_stream(device).cuda_stream)
    if key not in _SIDE:
        _SIDE[key] = torch.cuda.Stream(device=device)
    return _SIDE[key]


def stage_forward(stage: StageModel, weights, key, x: torch.Tensor, version: int,
                  check_finite: bool = True, finite_flags: torch.Tensor | None = None,
                  flag_index: int = 0, loss_req: dict | None = None) -> torch.Tensor:
    """Run the stage's layers on x with the given weights view; stash the
    per-layer inputs and pre-activations (stages.py:156-184).

    check_finite=True raises NumericError immediately (host sync); otherwise,
    if `finite_flags` is given, a device-side all-finite bit is recorded at
    `flag_index` and checked later by the runtime.
    """
    if x.shape[1] != stage.in_dim:
        raise DimensionError(f"stage {stage.rank}: input has {x.shape[1]} cols, expected {stage.in_dim}")
    inputs, pres = [], []
    h = x
    fused = x.is_cuda
    checked = False
    side_check = None
    if fused and stage.rank == 0 and _tc_ok(x):
        # the tensor-core fp32 GEMM saturates a non-finite INPUT (its bf16 split
        # clamps +-inf) instead of propagating it to the output the reference
        # checks (stages.py:182); the data entering stage 0 is therefore checked
        # itself (later stages' inputs are earlier stages' checked outputs)
        if check_finite:
            if not bool(torch.isfinite(x).all()):
                raise NumericError(f"non-finite value in stage {stage.rank} forward output (non-finite input)")
        elif finite_flags is not None:
            # off the critical path: the check only reads x, so it runs on a
            # side stream beside the forward GEMMs and joins at the end
            side_check = _side_stream(x.device)
            fork = torch.cuda.Event()
            fork.record()
            side_check.wait_event(fork)
            with torch.cuda.stream(side_check):
                record_finite(x, finite_flags, flag_index)
    last = len(stage.layers) - 1
    for i, spec in enumerate(stage.layers):
        w, b = weights[2 * i], weights[2 * i + 1]
        inputs.append(h)
        if fused:
            # split-K GEMM + one reduce/bias/activation launch (which also
            # writes the deferred finiteness flag of the stage output), or bias
            # + ReLU in the cuBLASLt epilogue; relu layers stash relu(pre)
            want_flag = i == last and not check_finite and finite_flags is not None
            pre, h, checked = _affine(h, w, b, spec.activation, finite_flags if want_flag else None, flag_index,
                                      loss_req if i == last else None)
            pres.append(pre)
            continue
        pre = torch.addmm(b, h, w)
        pres.append(pre)
        h = _activate(pre, spec.activation)
    if check_finite:
        if not bool(torch.isfinite(h).all()):
            bad = torch.nonzero(~torch.isfinite(h))[0].tolist()
            raise NumericError(
                f"non-finite value in stage {stage.rank} forward output at entry ({bad[0]}, {bad[1]})"
            )
    elif finite_flags is not None and not checked:
        record_finite(h, finite_flags, flag_index)
    if side_check is not None:
        torch.cuda.current_stream(x.device).wait_stream(side_check)
    stage.stash.put(key, StashEntry(version, inputs, pres))
    return h


def record_finite(t: torch.Tensor, flags: torch.Tensor, index: int) -> None:
    """flags[index] = all(isfinite(t)) without a host sync: one po_all_finite
    launch on CUDA (flags must be pre-set to True)."""
    if t.is_cuda:
        from . import _lib

        tc = t if t.is_contiguous() else t.contiguous()
        rc = _lib.load().po_all_finite(tc.data_ptr(), tc.numel(), flags.data_ptr(), index,
                                       torch.cuda.current_stream(t.device).cuda_stream)
        _lib.check(rc, "po_all_finite")
    else:
        flags[index] = torch.isfinite(t).all()


# Weight gradients of MLP layers fused into the update that follows the
# backward (po_wgrad_update, a tcgen05 GEMM with K2/K3 in its epilogue):
# stage_backward(defer_wgrad=True) leaves those layers' dW uncomputed and
# records (param index, x, dpre) in stage.deferred_wgrad for
# OptimizerState.step_fused_. Off by default: 10-16 % faster than the
# split-K GEMM + K3 per stage at config 1's shapes, but in the 1F1B run it
# raises the prediction overhead (csrc/pipeoptim_wgrad.cu header,
# profiles/r2_wgrad_fused_bench.jsonl); True runs it (tests cover both).
FUSE_WGRAD_UPDATE = False


def _wgrad_fusable(x: torch.Tensor, dpre: torch.Tensor, gw: torch.Tensor) -> bool:
    from . import _lib

    return (x.is_cuda and x.dtype == torch.float32 and dpre.dtype == torch.float32 and x.is_contiguous()
            and dpre.is_contiguous() and gw.is_contiguous() and x.data_ptr() % 16 == 0 and dpre.data_ptr() % 16 == 0
            and gw.data_ptr() % 32 == 0
            and _lib.load().po_wgrad_update_supported(x.shape[0], x.shape[1], dpre.shape[1]) == 1)


def stage_backward(stage: StageModel, weights, key, grad_out: torch.Tensor,
                   accumulate: bool = False, need_input_grad: bool = True, defer_wgrad: bool = False):
    """Backpropagate through the stash (stages.py:187-209). Parameter grads go
    into stage.flat.grad's views (overwritten, or added when `accumulate`);
    the input gradient uses `weights` — the view at BACKWARD time.
    Returns (grad wrt stage input or None, list of parameter-grad views).

    On the device an input gradient that feeds a ReLU layer stays as its
    split-K partial products: po_relu_bwd_bias sums them (fixed order) in the
    same launch that applies the ReLU mask and forms the bias gradient.

    defer_wgrad (the caller runs the stage's update next, nothing reads the
    gradient in between): the weight gradients of the ReLU / linear layers
    whose shapes po_wgrad_update handles are not computed here; their
    (param index, x, dpre) go to stage.deferred_wgrad for
    OptimizerState.step_fused_, which forms them on the tensor cores inside
    the update."""
    entry = stage.stash.pop(key)
    stage.deferred_wgrad = []
    gviews = stage.flat.grads
    if not grad_out.is_cuda:
        return _stage_backward_host(stage, entry, weights, gviews, grad_out, accumulate, need_input_grad)
    from . import _lib

    lib = _lib.load()
    stream = torch.cuda.current_stream(grad_out.device).cuda_stream
    g = (grad_out if grad_out.is_contiguous() else grad_out.contiguous()).unsqueeze(0)  # [splits, rows, cols]
    for i in reversed(range(len(stage.layers))):
        spec = stage.layers[i]
        x = entry.layer_inputs[i]
        gw, gb = gviews[2 * i], gviews[2 * i + 1]
        if spec.activation == "linear" and g.shape[0] == 1 and _head_ok(x, weights[2 * i], "linear") \
                and gw.is_contiguous():
            # narrow linear layer: dx, dW, db in one launch (po_head_bwd)
            rows = x.shape[0]
            need = i > 0 or need_input_grad
            dx = torch.empty((rows, x.shape[1]), dtype=torch.float32, device=g.device) if need else None
            xc = x if x.is_contiguous() else x.contiguous()
            gc = g[0] if g[0].is_contiguous() else g[0].contiguous()
            rc = lib.po_head_bwd(xc.data_ptr(), rows, x.shape[1], gc.data_ptr(), gw.shape[1],
                                 weights[2 * i].data_ptr(), None if dx is None else dx.data_ptr(), gw.data_ptr(),
                                 gb.data_ptr(), int(accumulate), stream)
            _lib.check(rc, "po_head_bwd")
            g = None if dx is None else dx.unsqueeze(0)
            continue
        if spec.activation in ("relu", "linear"):
            # sum of the partials, dpre = g * act'(pre) and db = colsum(dpre) in one launch
            splits, rows, cols = g.shape
            dpre = torch.empty((rows, cols), dtype=torch.float32, device=g.device)
            relu = spec.activation == "relu"
            rc = lib.po_act_bwd_bias(int(relu), g.data_ptr(), splits, entry.pre_acts[i].data_ptr() if relu else None,
                                     rows, cols, dpre.data_ptr(), gb.data_ptr(), int(accumulate), stream)
            _lib.check(rc, "po_act_bwd_bias")
            if defer_wgrad and not accumulate and FUSE_WGRAD_UPDATE and _wgrad_fusable(x, dpre, gw):
                stage.deferred_wgrad.append((2 * i, x, dpre))
            else:
                _weight_grad(x, dpre, gw, accumulate)
        else:
            gfull = g[0] if g.shape[0] == 1 else _splitk_reduce(g, None, "linear")
            dpre = _activation_grad_mul(gfull, entry.pre_acts[i], spec.activation)
            if accumulate:
                gw.addmm_(x.t(), dpre)
                gb.add_(dpre.sum(dim=0, keepdim=True))
            else:
                torch.mm(x.t(), dpre, out=gw)
                torch.sum(dpre, dim=0, keepdim=True, out=gb)
        if i > 0 or need_input_grad:
            g = _input_grad_parts(dpre, weights[2 * i])
        else:
            g = None
    if g is not None:
        g = g[0] if g.shape[0] == 1 else _splitk_reduce(g, None, "linear")
    return g, gviews


def _stage_backward_host(stage, entry, weights, gviews, g, accumulate, need_input_grad):
    """CPU tensors (the gloo tests of the distributed runner): plain torch."""
    for i in reversed(range(len(stage.layers))):
        spec = stage.layers[i]
        x = entry.layer_inputs[i]
        gw, gb = gviews[2 * i], gviews[2 * i + 1]
        dpre = _activation_grad_mul(g, entry.pre_acts[i], spec.activation)
        if accumulate:
            gw.addmm_(x.t(), dpre)
            gb.add_(dpre.sum(dim=0, keepdim=True))
        else:
            torch.mm(x.t(), dpre, out=gw)
            torch.sum(dpre, dim=0, keepdim=True, out=gb)
        g = torch.mm(dpre, weights[2 * i].t()) if (i > 0 or need_input_grad) else None
    return g, gviews


def network_forward(stages: list[StageModel], params_per_stage, x: torch.Tensor) -> torch.Tensor:
    """Chained forward over all stages with explicit weights; no stash (stages.py:212-218)."""
    h = x
    for stage, weights in zip(stages, params_per_stage):
        for i, spec in enumerate(stage.layers):
            h = _activate(torch.addmm(weights[2 * i + 1], h, weights[2 * i]), spec.activation)
    return h


def params_by_layer(stages: list[StageModel]) -> dict[int, tuple[torch.Tensor, torch.Tensor]]:
    """Live (w, b) per global layer index, partition independent (stages.py:221-227)."""
    out = {}
    for stage in stages:
        p = stage.params
        for i, spec in enumerate(stage.layers):
            out[spec.index] = (p[2 * i], p[2 * i + 1])
    return out


# ---- losses (linalg.py:212-241) ----------------------------------------------------------------

LOSS_KINDS = ("mse", "softmax_xent")


_LOSS_SCRATCH: dict = {}


def loss_and_grad(pred: torch.Tensor, target: torch.Tensor, kind: str):
    """(loss as a 0-d device tensor, grad wrt pred).

    mse: mean over all entries of (pred - target)^2, grad 2*(pred - target)/numel.
    softmax_xent: logits vs one-hot target, row-max-shifted softmax, mean row
    cross-entropy, grad (softmax - target)/rows.
    On CUDA this is ONE fused launch (po_loss_grad); on CPU (the gloo tests
    of the distributed runner) plain torch ops.
    """
    if pred.shape != target.shape:
        raise DimensionError(f"loss_and_grad: shapes differ: {tuple(pred.shape)} vs {tuple(target.shape)}")
    if kind not in LOSS_KINDS:
        raise ValueError(f"unknown loss kind: {kind!r}")
    if pred.is_cuda and pred.dim() == 2:
        from . import _lib

        rows, cols = pred.shape
        p = pred if pred.is_contiguous() else pred.contiguous()
        t = target.to(torch.float32)
        t = t if t.is_contiguous() else t.contiguous()
        stream = torch.cuda.current_stream(pred.device).cuda_stream
        # scratch (row partials + the last-CTA counter) per device, row count
        # and stream: launches on different streams must not share a counter
        key = (pred.device, rows, stream)
        if key not in _LOSS_SCRATCH:
            _LOSS_SCRATCH[key] = torch.zeros(rows + 1, dtype=torch.float32, device=pred.device)
        grad = torch.empty_like(p)
        loss = torch.empty((), dtype=torch.float32, device=pred.device)
        code = _lib.PO_LOSS_MSE if kind == "mse" else _lib.PO_LOSS_SOFTMAX_XENT
        rc = _lib.load().po_loss_grad(code, p.data_ptr(), t.data_ptr(), rows, cols, grad.data_ptr(),
                                      loss.data_ptr(), _LOSS_SCRATCH[key].data_ptr(), stream)
        _lib.check(rc, "po_loss_grad")
        return loss, grad
    if kind == "mse":
        diff = pred - target
        n = diff.numel()
        loss = (diff * diff).sum() / n
        grad = 2.0 * diff / n
    elif kind == "softmax_xent":
        z = pred - pred.max(dim=1, keepdim=True).values
        ez = torch.exp(z)
        sm = ez / ez.sum(dim=1, keepdim=True)
        picked = (sm * target).sum(dim=1)
        loss = (-torch.log(picked)).mean()
        grad = (sm - target) / pred.shape[0]
    else:
        raise ValueError(f"unknown loss kind: {kind!r}")
    return loss, grad
