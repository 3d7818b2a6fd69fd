"""Pipeline stages built from torch modules (configs 2-4: VGG-16, ResNet-101,
GNMT-style LSTM), with the reference's weight-view semantics.

The reference only has dense MLP stages (stages.py); BASELINE configs 2-4 are
deep models, so here a stage is a contiguous slice of a model's blocks whose
parameters are re-pointed (`param.data = view`) into the stage's flat fp32
buffer (FlatParams) and whose `.grad`s are views of the flat gradient — so
the predictor/optimizer kernels stream the whole stage in one launch exactly
as for the MLP stages, and the same runners drive both.

Forward/backward semantics (stages.py:156-209): the forward
runs on the policy's view (W_hat for predicted stages) by pointing every
parameter's storage at the staging buffer for the duration of the forward;
the backward runs after the parameters point back at the LIVE buffer.
Convolution and batch-norm autograd nodes save the parameter object itself,
so their input gradients use the live weights at backward time, as the
reference does; `nn.Linear` would save a transposed view of the forward-time
storage, so linear layers use `LiveLinear`, whose backward reads the live
weight explicitly; LSTM layers use `LiveLSTM` (cuBLAS GEMMs + the
po_lstm_cell_fwd/bwd kernels), whose backward propagates through the live
weights (cuDNN's LSTM would keep its own packed forward-time copy).

Exception — the bf16-autocast variant (`amp_dtype`, a throughput-only arm of
the bench): autocast casts each conv weight to a fresh bf16 tensor, and the
convolution's autograd node saves THAT copy, so conv input gradients go
through the forward-time (predicted) weights, not the live ones. Linear
layers keep the live-weight rule. The amp arm therefore does not carry the
S9 semantics and is excluded from every parity claim; the fp32 path does.

Image stages can run NHWC inside the stage (`channels_last=True`; boundary
tensors stay NCHW), and their batch norms run on PyTorch's native kernels:
cuDNN's training batch-norm kernels synchronise across their grid and can
deadlock when two stages run concurrently on one GPU (runtime streams="stage").
"""

from __future__ import annotations

import math

import torch
import torch.nn as nn
import torch.nn.functional as F

from . import _lib
from .errors import NumericError
from .optim import FlatParams
from .stages import ActivationStash, StashEntry, _splitk, loss_and_grad, record_finite


class _LiveLinearFn(torch.autograd.Function):
    """y = x W^T + b; backward: dx = g W_live, dW = g^T x, db = colsum(g).
    `dt` (autocast): the forward computes in dt from dt casts of x, W, b; the
    backward multiplies by the LIVE weight cast to dt; autograd returns the
    parameter gradients to the fp32 flat buffer in fp32."""

    @staticmethod
    def forward(ctx, x, weight, bias, module, dt=None):
        ctx.save_for_backward(x)
        ctx.module, ctx.dt = module, dt
        if dt is not None:
            return F.linear(x, weight.to(dt), None if bias is None else bias.to(dt))
        return F.linear(x, weight, bias)

    @staticmethod
    def backward(ctx, g):
        (x,) = ctx.saved_tensors
        w_live = ctx.module.weight  # points at the live buffer again by now
        if ctx.dt is not None:
            w_live = w_live.to(ctx.dt)
        gx = g.matmul(w_live)
        g2 = g.reshape(-1, g.shape[-1])
        x2 = x.reshape(-1, x.shape[-1])
        gw = g2.t().matmul(x2)
        gb = g2.sum(0) if ctx.module.bias is not None else None
        return gx, gw, gb, None, None


class LiveLinear(nn.Linear):
    def forward(self, x):
        if x.is_cuda and torch.is_autocast_enabled("cuda"):
            dt = torch.get_autocast_dtype("cuda")
            with torch.autocast("cuda", enabled=False):
                return _LiveLinearFn.apply(x.to(dt), self.weight, self.bias, self, dt)
        return _LiveLinearFn.apply(x, self.weight, self.bias, self)


# ---- model definitions (as lists of blocks for contiguous partitioning) ------------------


def vgg16_cifar_blocks(num_classes: int = 100) -> list[nn.Module]:
    """VGG-16 for 32x32 inputs (conv3x3-BN-ReLU x13, 5 max-pools, 512-512-C
    classifier): ~15.3M params."""
    cfg = [64, 64, "M", 128, 128, "M", 256, 256, 256, "M", 512, 512, 512, "M", 512, 512, 512, "M"]
    blocks: list[nn.Module] = []
    c_in = 3
    pending = []
    for v in cfg:
        if v == "M":
            pending.append(nn.MaxPool2d(2, 2))
            blocks.append(nn.Sequential(*pending))
            pending = []
        else:
            if pending:
                blocks.append(nn.Sequential(*pending))
            pending = [nn.Conv2d(c_in, v, 3, padding=1, bias=False), nn.BatchNorm2d(v), nn.ReLU(inplace=True)]
            c_in = v
    blocks.append(nn.Sequential(nn.Flatten(), LiveLinear(512, 512), nn.ReLU(inplace=True)))
    blocks.append(nn.Sequential(LiveLinear(512, 512), nn.ReLU(inplace=True), LiveLinear(512, num_classes)))
    return blocks


def resnet101_blocks(num_classes: int = 200) -> list[nn.Module]:
    """torchvision ResNet-101 (bottleneck 3-4-23-3) as stem, 33 bottlenecks,
    head; 42.9M params at 200 classes."""
    import torchvision

    m = torchvision.models.resnet101(weights=None, num_classes=num_classes)
    fc = LiveLinear(m.fc.in_features, num_classes)
    blocks: list[nn.Module] = [nn.Sequential(m.conv1, m.bn1, m.relu, m.maxpool)]
    for layer in (m.layer1, m.layer2, m.layer3, m.layer4):
        blocks.extend(list(layer))
    blocks.append(nn.Sequential(m.avgpool, nn.Flatten(), fc))
    return blocks


class _LiveLSTMFn(torch.autograd.Function):
    """One batch-first LSTM layer (PyTorch gate order i, f, g, o) with the
    reference's stage semantics (stages.py:187-209, S9): the forward runs on
    the weights it is given (W_hat for a predicted stage) and stashes its
    activations; the backward forms dW from those activations and propagates
    dx / dh through the LIVE weights (the module's parameters at backward
    time), exactly as the MLP stage's `g = dpre W_live^T`.

    Layout: time-major inside (x^T (T, B, Din), gates (T, B, 4H), h (T+1, B, H),
    c (T, B, H)), batch-first at the boundary. Forward: one GEMM for all
    input projections, then per step one split-K batched GEMM (h_{t-1}
    W_hh^T) and one po_lstm_cell_fwd_sk that sums its partials into the
    gates. Backward: per step one po_lstm_cell_bwd_sk (summing the partials
    of dh) and one split-K GEMM (dh_{t-1} = dgates_t W_hh_live), then three
    GEMMs over all steps (dx, dW_ih, dW_hh) and a column sum (db)."""

    @staticmethod
    def forward(ctx, x, w_ih, w_hh, b_ih, b_hh, module):
        if not x.is_cuda:
            raise RuntimeError("LiveLSTM runs on the B200 kernels (po_lstm_cell_*): no CPU path")
        lib = _lib.load()
        stream = torch.cuda.current_stream(x.device).cuda_stream
        bsz, steps, d_in = x.shape
        hid = w_hh.shape[1]
        xt = x.detach().transpose(0, 1).contiguous()
        gates = torch.addmm(b_ih + b_hh, xt.view(steps * bsz, d_in), w_ih.t()).view(steps, bsz, 4 * hid)
        hs = torch.empty((steps + 1, bsz, hid), device=x.device, dtype=x.dtype)
        cs = torch.empty((steps, bsz, hid), device=x.device, dtype=x.dtype)
        y = torch.empty((bsz, steps, hid), device=x.device, dtype=x.dtype)
        w_hh_t = w_hh.t()
        # the recurrent GEMM (batch x H @ H x 4H) has few output tiles: run it
        # split-K and let the cell kernel sum the partials (po_lstm_cell_fwd_sk)
        sk = _splitk(bsz, hid, 4 * hid) if module.split_k else 1
        if sk > 1:
            w_split = w_hh.view(4 * hid, sk, hid // sk).permute(1, 2, 0)  # (S, H/S, 4H) slices of W_hh^T
            part = torch.empty((sk, bsz, 4 * hid), device=x.device, dtype=x.dtype)
        for t in range(steps):
            rec = None
            if t > 0:
                if sk > 1:
                    torch.bmm(hs[t].view(bsz, sk, hid // sk).transpose(0, 1), w_split, out=part)
                    rec = part.data_ptr()
                else:
                    gates[t].addmm_(hs[t], w_hh_t)
            rc = lib.po_lstm_cell_fwd_sk(gates[t].data_ptr(), rec, sk, cs[t - 1].data_ptr() if t else None,
                                         cs[t].data_ptr(), hs[t + 1].data_ptr(), y[:, t].data_ptr(), steps * hid, bsz,
                                         hid, stream)
            _lib.check(rc, "po_lstm_cell_fwd_sk")
        ctx.save_for_backward(xt, gates, hs, cs)
        ctx.module = module
        return y

    @staticmethod
    def backward(ctx, dy):
        xt, gates, hs, cs = ctx.saved_tensors
        m = ctx.module
        w_ih, w_hh = m.weight_ih_l0, m.weight_hh_l0  # point at the live buffer again by now
        lib = _lib.load()
        stream = torch.cuda.current_stream(dy.device).cuda_stream
        steps, bsz, hid4 = gates.shape
        hid = hid4 // 4
        d_in = xt.shape[2]
        dy = dy.contiguous()
        dg = torch.empty_like(gates)
        dc = torch.zeros((bsz, hid), device=dy.device, dtype=dy.dtype)
        # dh_{t-1} = dgates_t W_hh_live (batch x 4H @ 4H x H): split-K, the
        # partials summed inside po_lstm_cell_bwd_sk
        sk = _splitk(bsz, hid4, hid) if m.split_k else 1
        w_split = w_hh.view(sk, hid4 // sk, hid)
        ping = torch.empty((2, sk, bsz, hid), device=dy.device, dtype=dy.dtype)
        rec = None
        for t in range(steps - 1, -1, -1):
            rc = lib.po_lstm_cell_bwd_sk(gates[t].data_ptr(), cs[t - 1].data_ptr() if t else None, cs[t].data_ptr(),
                                         dy[:, t].data_ptr(), steps * hid, rec, sk, dc.data_ptr(), dg[t].data_ptr(),
                                         bsz, hid, stream)
            _lib.check(rc, "po_lstm_cell_bwd_sk")
            if t > 0:
                buf = ping[t % 2]
                if sk > 1:
                    torch.bmm(dg[t].view(bsz, sk, hid4 // sk).transpose(0, 1), w_split, out=buf)
                else:
                    torch.mm(dg[t], w_hh, out=buf[0])
                rec = buf.data_ptr()
        dg2 = dg.view(steps * bsz, hid4)
        dx = None
        if ctx.needs_input_grad[0]:
            dx = torch.mm(dg2, w_ih).view(steps, bsz, d_in).transpose(0, 1)
        gw_ih = dg2.t().mm(xt.view(steps * bsz, d_in))
        if steps > 1:  # h_{-1} = 0 contributes nothing
            gw_hh = dg[1:].reshape((steps - 1) * bsz, hid4).t().mm(hs[1:steps].reshape((steps - 1) * bsz, hid))
        else:
            gw_hh = torch.zeros_like(w_hh)
        gb = dg2.sum(0)
        return dx, gw_ih, gw_hh, gb, gb, None


class LiveLSTM(nn.Module):
    """Single-layer batch-first LSTM with nn.LSTM's parameters, names and
    initialisation (weight_ih_l0, weight_hh_l0, bias_ih_l0, bias_hh_l0, each
    U(-1/sqrt(H), 1/sqrt(H)) in that order) whose backward uses the live
    weights (see _LiveLSTMFn). forward(x) -> (y, None)."""

    def __init__(self, input_size: int, hidden_size: int):
        super().__init__()
        self.input_size, self.hidden_size = input_size, hidden_size
        # split-K recurrent GEMMs: lower latency per step (a stage alone on its
        # GPU, the pipeline's critical path) at more SM-time per step; stages
        # sharing one GPU concurrently prefer the unsplit GEMMs (set_lstm_split_k)
        self.split_k = True
        h4 = 4 * hidden_size
        self.weight_ih_l0 = nn.Parameter(torch.empty(h4, input_size))
        self.weight_hh_l0 = nn.Parameter(torch.empty(h4, hidden_size))
        self.bias_ih_l0 = nn.Parameter(torch.empty(h4))
        self.bias_hh_l0 = nn.Parameter(torch.empty(h4))
        stdv = 1.0 / math.sqrt(hidden_size)
        for w in (self.weight_ih_l0, self.weight_hh_l0, self.bias_ih_l0, self.bias_hh_l0):
            nn.init.uniform_(w, -stdv, stdv)

    def forward(self, x):
        return _LiveLSTMFn.apply(x, self.weight_ih_l0, self.weight_hh_l0, self.bias_ih_l0, self.bias_hh_l0,
                                 self), None


def set_lstm_split_k(stages, flag: bool) -> None:
    """Latency (split-K, one stage per GPU) or SM-time (unsplit, stages
    sharing a GPU) recurrent GEMMs for every LiveLSTM of the stages."""
    for st in stages:
        for m in st.module.modules():
            if isinstance(m, LiveLSTM):
                m.split_k = flag


class _LSTMBlock(nn.Module):
    def __init__(self, d_in, d, residual):
        super().__init__()
        self.lstm = LiveLSTM(d_in, d)
        self.residual = residual

    def forward(self, x):
        y, _ = self.lstm(x)
        return y + x if self.residual else y


class _Embed(nn.Module):
    def __init__(self, vocab, d):
        super().__init__()
        self.emb = nn.Embedding(vocab, d)

    def forward(self, tokens):
        return self.emb(tokens.long())


class _Head(nn.Module):
    def __init__(self, d, vocab):
        super().__init__()
        self.proj = LiveLinear(d, vocab)

    def forward(self, x):
        return self.proj(x[:, -1, :])


def gnmt8_blocks(vocab: int = 32000, d: int = 1024) -> list[nn.Module]:
    """GNMT-8-shaped sequential stack: embedding, 8 LSTM layers of width d
    (residual from layer 3 on, as GNMT), projection to the vocabulary on the
    last position (the encoder/decoder attention is
    folded into a sequential stack so it partitions into a pipeline)."""
    blocks: list[nn.Module] = [_Embed(vocab, d)]
    for i in range(8):
        blocks.append(_LSTMBlock(d, d, residual=i >= 2))
    blocks.append(_Head(d, vocab))
    return blocks


def balanced_partition(costs: list[float], depth: int) -> list[tuple[int, int]]:
    """Contiguous split of blocks into `depth` non-empty ranges minimising the
    largest range cost (DP over prefix sums). Returns [(lo, hi)) ranges."""
    n = len(costs)
    if not 1 <= depth <= n:
        raise ValueError(f"cannot split {n} blocks across {depth} stages")
    pre = [0.0]
    for c in costs:
        pre.append(pre[-1] + c)
    INF = float("inf")
    best = [[INF] * (n + 1) for _ in range(depth + 1)]
    cut = [[0] * (n + 1) for _ in range(depth + 1)]
    best[0][0] = 0.0
    for k in range(1, depth + 1):
        for j in range(k, n - (depth - k) + 1):
            for i in range(k - 1, j):
                v = max(best[k - 1][i], pre[j] - pre[i])
                if v < best[k][j]:
                    best[k][j] = v
                    cut[k][j] = i
    out, j = [], n
    for k in range(depth, 0, -1):
        i = cut[k][j]
        out.append((i, j))
        j = i
    return out[::-1]


def block_param_counts(blocks: list[nn.Module]) -> list[int]:
    return [sum(p.numel() for p in b.parameters()) for b in blocks]


# ---- the stage --------------------------------------------------------------------------------


class _GridSafeBatchNorm2d(nn.BatchNorm2d):
    """BatchNorm2d on PyTorch's native kernels instead of cuDNN's.

    cuDNN's training-mode batch-norm kernels (`bn_fw_tr_1C11_singleread`,
    `batchnorm_fwtr_nhwc_semiPersist` and their backward twins) synchronise
    across their whole grid, sized for an otherwise idle GPU. When the
    stage-concurrent runner puts two such launches on different stage streams,
    each can hold SMs while it waits for CTAs that never become resident: a
    GPU deadlock (reproduced on the B200 with config 3 within ~6 runs). The
    native kernels reduce with a last-block pattern, which never waits for
    other CTAs to be co-resident. The autograd node is chosen at forward time,
    so the backward stays native too."""

    def forward(self, x):
        prev = torch.backends.cudnn.enabled
        torch.backends.cudnn.enabled = False
        try:
            return super().forward(x)
        finally:
            torch.backends.cudnn.enabled = prev


def _use_grid_safe_bn(module: nn.Module) -> None:
    for m in module.modules():
        if type(m) is nn.BatchNorm2d:
            m.__class__ = _GridSafeBatchNorm2d


def use_cudnn_bn(stages) -> None:
    """Put cuDNN's batch norm back on these stages: safe (and faster) where a
    stage's work is the only work on its GPU — one stage per GPU, or stages
    serialised on one stream — never with streams="stage"."""
    for st in stages:
        for m in st.module.modules():
            if type(m) is _GridSafeBatchNorm2d:
                m.__class__ = nn.BatchNorm2d


class ModuleStage:
    """A pipeline stage made of torch modules over a flat parameter buffer.

    Same surface the runners use on the MLP `StageModel`: rank, flat, params,
    param_names, version, stash, in_shape/out_shape (per sample) and
    run_forward / run_backward.
    """

    def __init__(self, rank: int, blocks: list[nn.Module], device, in_shape: tuple, in_dtype=torch.float32,
                 channels_last: bool = False, amp_dtype=None):
        """channels_last=True runs the stage's image tensors in NHWC inside the
        stage (cuDNN's native tensor-core layout); boundary activations and
        gradients stay NCHW-contiguous, so transports and the other stages are
        unaffected. Parameters keep their flat NCHW views either way.
        amp_dtype (e.g. torch.bfloat16): the stage's forward runs under
        autocast in that dtype (tensor-core convs/GEMMs); the parameters,
        gradients, optimizer state and boundary tensors stay fp32."""
        self.rank = rank
        self.channels_last = channels_last
        self.amp_dtype = amp_dtype
        self.device = torch.device(device)
        self.module = nn.Sequential(*blocks).to(self.device)
        self.module.train()
        _use_grid_safe_bn(self.module)
        named = list(self.module.named_parameters())
        self._params = [p for _, p in named]
        self.param_names = [n for n, _ in named]
        self.flat = FlatParams.from_tensors(self.param_names, [p.detach() for p in self._params], self.device)
        self._live = self.flat.params
        for p, v, gv in zip(self._params, self._live, self.flat.grads):
            p.data = v
            p.grad = gv
        self.version = 1
        self.stash = ActivationStash()
        self.in_shape = tuple(in_shape)
        self.in_dtype = in_dtype
        with torch.no_grad():
            probe = torch.zeros((2, *self.in_shape), device=self.device, dtype=in_dtype)
            self.out_shape = tuple(self.module(probe).shape[1:])
        # the probe ran in train mode: reset batch-norm statistics it touched
        for m in self.module.modules():
            if isinstance(m, nn.modules.batchnorm._BatchNorm):
                m.reset_running_stats()

    @property
    def params(self) -> list[torch.Tensor]:
        return self._live

    @property
    def numel(self) -> int:
        return self.flat.layout.numel

    def set_grad_buffer(self, buf: torch.Tensor) -> None:
        self.flat.grad = buf
        for p, gv in zip(self._params, self.flat.grads):
            p.grad = gv

    def set_weight_buffer(self, buf: torch.Tensor) -> None:
        """Move the live weights into `buf` (same layout) and re-point the
        module's parameters at it."""
        buf.copy_(self.flat.data)
        self.flat.data = buf
        self._live = self.flat.params
        self._point(self._live)

    def _point(self, views) -> None:
        for p, v in zip(self._params, views):
            if p.data_ptr() != v.data_ptr():
                p.data = v

    def run_forward_loss(self, weights, key, x, version, target, loss_kind, check_finite=True, finite_flags=None,
                         flag_index=0):
        """Last-stage forward + loss (runtime.py:415-426): (out, loss, dL/dout)."""
        out = self.run_forward(weights, key, x, version, check_finite, finite_flags, flag_index)
        loss, grad = loss_and_grad(out, target, loss_kind)
        return out, loss, grad

    def run_forward(self, weights, key, x, version, check_finite=True, finite_flags=None, flag_index=0):
        self._point(weights)
        try:
            x_in = x.detach()
            if self.rank > 0 and x_in.is_floating_point():
                x_in.requires_grad_(True)
            with torch.enable_grad():
                h = x_in
                if self.channels_last and h.dim() == 4:
                    h = h.contiguous(memory_format=torch.channels_last)
                if self.amp_dtype is not None:
                    # no cast cache: the parameters are re-pointed every forward
                    # (and the forward may be captured into a CUDA graph)
                    with torch.autocast("cuda", dtype=self.amp_dtype, cache_enabled=False):
                        out = self.module(h)
                    out = out.float()
                else:
                    out = self.module(h)
                if not out.is_contiguous():
                    out = out.contiguous()
        finally:
            self._point(self._live)
        if check_finite:
            if not bool(torch.isfinite(out).all()):
                raise NumericError(f"non-finite value in stage {self.rank} forward output")
        elif finite_flags is not None:
            record_finite(out, finite_flags, flag_index)
        self.stash.put(key, StashEntry(version, [x_in], [out]))
        return out.detach()

    def run_backward(self, weights, key, grad_out, accumulate=False, need_input_grad=True):
        entry = self.stash.pop(key)
        x_in, out = entry.layer_inputs[0], entry.pre_acts[0]
        self._point(weights)
        try:
            if not accumulate:
                self.flat.grad.zero_()
            torch.autograd.backward(out, grad_out)
        finally:
            self._point(self._live)
        g_in = x_in.grad if (need_input_grad and x_in.requires_grad) else None
        return g_in, self.flat.grads


def profile_block_costs(blocks, in_shape, batch, device, in_dtype=torch.float32, reps=7,
                        channels_last: bool = False, warmup: int = 2) -> list[float]:
    """Per-block forward+backward time on the device for one batch (a tiny
    profiling partitioner, in the spirit of PipeDream's), used to balance
    stages by time instead of parameter count."""
    dev = torch.device(device)
    x = torch.zeros((batch, *in_shape), device=dev, dtype=in_dtype)
    if in_dtype == torch.float32:
        x.normal_()
    if channels_last and x.dim() == 4:
        x = x.contiguous(memory_format=torch.channels_last)
    costs = []
    for b in blocks:
        b.to(dev).train()
        xin = x.detach().requires_grad_(x.is_floating_point())
        _use_grid_safe_bn(b)  # profile the kernels the stages will run
        for _ in range(warmup):  # cuDNN/cuBLAS algorithm selection, lazy allocations
            y = b(xin)
            y.backward(torch.ones_like(y))
        times = []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            y = b(xin)
            y.backward(torch.ones_like(y))
            e1.record()
            e1.synchronize()
            times.append(e0.elapsed_time(e1))
        b.zero_grad(set_to_none=True)
        costs.append(sorted(times)[len(times) // 2])
        x = y.detach()
    for m in (mm for b in blocks for mm in b.modules()):
        if isinstance(m, nn.modules.batchnorm._BatchNorm):
            m.reset_running_stats()
    return costs


def build_module_stages(blocks, depth, device, in_shape, costs=None, in_dtype=torch.float32,
                        channels_last: bool = False, amp_dtype=None):
    """Partition `blocks` into `depth` contiguous stages balanced by `costs`
    (default: parameter counts) and build them in order."""
    costs = costs if costs is not None else [max(1, c) for c in block_param_counts(blocks)]
    ranges = balanced_partition(costs, depth)
    stages, shape, dtype = [], tuple(in_shape), in_dtype
    for k, (lo, hi) in enumerate(ranges):
        st = ModuleStage(k, blocks[lo:hi], device, shape, dtype, channels_last=channels_last, amp_dtype=amp_dtype)
        stages.append(st)
        shape, dtype = st.out_shape, torch.float32
    return stages
