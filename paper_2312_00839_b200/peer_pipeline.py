"""One-process-per-GPU 1F1B runner whose boundary tensors move by peer-memory
stores (NVLink / NVSwitch) instead of host-driven NCCL calls, so a rank's
whole run is one stream of device work — captured into ONE CUDA graph and
replayed with no host involvement.

Same program, policies, version bookkeeping and kernels as the NCCL runner
(`pipeline.PipelineStageRunner`): rank k executes `stage_program(tl, k)`,
i.e. the reference's `tl.stage_events(k)` order (pkg/src/pipesim/
schedule.py:80-81), which the reference simulates in one thread with
hand-off dicts (runtime.py:390-391, 420-433). Here each hand-off direction
of a boundary is a ring on the receiving GPU (csrc/pipeoptim_p2p.cu):
`po_p2p_send` stores the tensor into the peer's ring slot and release-stores
the peer's ready counter; `po_p2p_recv` waits for it, copies the slot into a
fresh input buffer (kept by the stash until the backward) and release-stores
the sender's ack counter (ring credit).

Deadlock freedom: a ring has `slots` = 1 + the most messages ever in flight
on that link in the reference's global event order (`ring_slots`). Then the
globally-earliest pending op of any blocked configuration can always
proceed — its message was produced earlier in that order, and the credit it
needs was returned earlier in it — so ranks never wait on each other in a
cycle.
"""

from __future__ import annotations

import math
import time

import torch

from . import _lib
from .errors import NumericError
from .ipc import IpcBuffer, open_peer
from .optim import CoefTape, MbLr
from .pipeline import StageReport
from .runtime import (
    PREDICTIVE_STRATEGIES,
    STRATEGY_SCHEDULE,
    VersionRecord,
    _make_policy,
    _StageRt,
    _to_device,
    capture,
    staging_in_grad_ok,
)
from .schedule import BACKWARD, FORWARD, UPDATE, Timeline, stage_program, validate_timeline

# flag word offsets in each rank's int64 flag block
_ACT_READY, _GRAD_READY, _ACT_ACK, _GRAD_ACK = 0, 1, 2, 3


def ring_slots(tl: Timeline) -> dict[tuple[str, int], int]:
    """1 + the most messages simultaneously in flight per link in the global
    event order: ("act", k) is stage k -> k+1 (produced by F(m, k), consumed
    by F(m, k+1)); ("grad", k) is stage k+1 -> k (B(m, k+1) -> B(m, k))."""
    live: dict[tuple[str, int], int] = {}
    peak: dict[tuple[str, int], int] = {}

    def bump(key, d):
        live[key] = live.get(key, 0) + d
        peak[key] = max(peak.get(key, 0), live[key])

    for e in tl.events:
        if e.kind == FORWARD:
            if e.stage > 0:
                bump(("act", e.stage - 1), -1)
            if e.stage < tl.depth - 1:
                bump(("act", e.stage), +1)
        elif e.kind == BACKWARD:
            if e.stage < tl.depth - 1:
                bump(("grad", e.stage), -1)
            if e.stage > 0:
                bump(("grad", e.stage - 1), +1)
    return {k: v + 1 for k, v in peak.items()}


def _slot_elems(rows: int, shape: tuple) -> int:
    n = rows * math.prod(shape)
    return (n + 63) // 64 * 64  # 256-byte aligned slots


class PeerLinks:
    """This rank's rings, flags and control blocks, and its neighbours' peer
    mappings (CUDA IPC handles exchanged with one object all-gather)."""

    def __init__(self, dist, rank: int, depth: int, rows: int, in_shape: tuple, out_shape: tuple, slots: dict,
                 device, group=None, stage_ranks: list[int] | None = None, timeout_ms: int = 60_000):
        self.rank, self.depth, self.device = rank, depth, torch.device(device)
        self.timeout_ms = timeout_ms
        self.in_elems = rows * math.prod(in_shape)
        self.out_elems = rows * math.prod(out_shape)
        self.in_shape, self.out_shape, self.rows = tuple(in_shape), tuple(out_shape), rows
        dev = self.device
        self._flags_buf = IpcBuffer(4, torch.int64, dev)  # written by the neighbours
        self.flags = self._flags_buf.tensor
        self.ctl_act = torch.zeros(4, dtype=torch.int64, device=dev)   # [sent to k+1, arr, recvd from k-1, arr]
        self.ctl_grad = torch.zeros(4, dtype=torch.int64, device=dev)  # [sent to k-1, arr, recvd from k+1, arr]
        self.status = torch.zeros(1, dtype=torch.int32, device=dev)
        # rings this rank RECEIVES into (stage k-1's activations, stage k+1's
        # gradients) and the geometry of the neighbours' rings it SENDS into
        # (same rule on both sides: the receiver's in_shape is the sender's out_shape)
        self.act_slots = slots.get(("act", rank - 1), 1)
        self.grad_slots = slots.get(("grad", rank), 1)
        self.act_slot_elems = _slot_elems(rows, in_shape)
        self.grad_slot_elems = _slot_elems(rows, out_shape)
        self.next_act_slots = slots.get(("act", rank), 1)
        self.next_act_slot_elems = _slot_elems(rows, out_shape)
        self.prev_grad_slots = slots.get(("grad", rank - 1), 1)
        self.prev_grad_slot_elems = _slot_elems(rows, in_shape)
        self._rings = [IpcBuffer(self.act_slots * self.act_slot_elems, torch.float32, dev) if rank > 0 else None,
                       IpcBuffer(self.grad_slots * self.grad_slot_elems, torch.float32, dev)
                       if rank < depth - 1 else None]
        self.act_ring = None if self._rings[0] is None else self._rings[0].tensor
        self.grad_ring = None if self._rings[1] is None else self._rings[1].tensor
        torch.cuda.synchronize(dev)
        mine = (self._flags_buf.export(), *(None if b is None else b.export() for b in self._rings))
        world = dist.get_world_size(group) if group is not None else dist.get_world_size()
        handles = [None] * world
        dist.all_gather_object(handles, mine, group=group)
        ranks = stage_ranks or list(range(depth))
        self._peers = []

        def open_(h):
            pb = open_peer(h, dev)
            self._peers.append(pb)
            return pb.tensor

        self.next = self.prev = None
        err = None
        try:
            if rank < depth - 1:
                h = handles[ranks[rank + 1]]
                self.next = (open_(h[0]), open_(h[1]))  # (flags, act_ring) of stage k+1
            if rank > 0:
                h = handles[ranks[rank - 1]]
                self.prev = (open_(h[0]), open_(h[2]))  # (flags, grad_ring) of stage k-1
        except Exception as exc:  # every rank must learn of it, or the group desynchronises
            err = exc
        self._lib = _lib.load()
        ok = torch.tensor([0 if err else 1], dtype=torch.int32,
                          device=dev if dist.get_backend(group) == "nccl" else "cpu")
        dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=group)
        if int(ok.item()) == 0:
            raise RuntimeError(f"peer mapping failed on a rank of the pipeline (here: {err!r})")

    def _flag(self, t: torch.Tensor, word: int) -> int:
        return t.data_ptr() + 8 * word

    def send_act(self, out: torch.Tensor) -> None:
        """Activation of this stage's forward -> stage k+1's ring."""
        flags, ring = self.next
        self._check_shape(out, self.out_elems)
        rc = self._lib.po_p2p_send(out.data_ptr(), out.numel(), ring.data_ptr(), self.next_act_slot_elems,
                                   self.next_act_slots, self.ctl_act.data_ptr(), self._flag(self.flags, _ACT_ACK),
                                   self._flag(flags, _ACT_READY), self.timeout_ms, self.status.data_ptr(),
                                   _stream(self.device))
        _lib.check(rc, "po_p2p_send")

    def recv_act(self) -> torch.Tensor:
        flags, _ = self.prev
        buf = torch.empty((self.rows, *self.in_shape), dtype=torch.float32, device=self.device)
        rc = self._lib.po_p2p_recv(self.act_ring.data_ptr(), self.act_slot_elems, self.act_slots, buf.data_ptr(),
                                   buf.numel(), self.ctl_act.data_ptr(), self._flag(self.flags, _ACT_READY),
                                   self._flag(flags, _ACT_ACK), self.timeout_ms, self.status.data_ptr(),
                                   _stream(self.device))
        _lib.check(rc, "po_p2p_recv")
        return buf

    def send_grad(self, g: torch.Tensor) -> None:
        """Input gradient of this stage's backward -> stage k-1's ring."""
        flags, ring = self.prev
        self._check_shape(g, self.in_elems)
        rc = self._lib.po_p2p_send(g.data_ptr(), g.numel(), ring.data_ptr(), self.prev_grad_slot_elems,
                                   self.prev_grad_slots, self.ctl_grad.data_ptr(), self._flag(self.flags, _GRAD_ACK),
                                   self._flag(flags, _GRAD_READY), self.timeout_ms, self.status.data_ptr(),
                                   _stream(self.device))
        _lib.check(rc, "po_p2p_send")

    def recv_grad(self) -> torch.Tensor:
        flags, _ = self.next
        buf = torch.empty((self.rows, *self.out_shape), dtype=torch.float32, device=self.device)
        rc = self._lib.po_p2p_recv(self.grad_ring.data_ptr(), self.grad_slot_elems, self.grad_slots, buf.data_ptr(),
                                   buf.numel(), self.ctl_grad.data_ptr(), self._flag(self.flags, _GRAD_READY),
                                   self._flag(flags, _GRAD_ACK), self.timeout_ms, self.status.data_ptr(),
                                   _stream(self.device))
        _lib.check(rc, "po_p2p_recv")
        return buf

    @staticmethod
    def _check_shape(t: torch.Tensor, n: int) -> None:
        if t.numel() != n or not t.is_contiguous() or t.dtype != torch.float32:
            raise ValueError(f"boundary tensor must be contiguous fp32 with {n} elements, got {tuple(t.shape)}")

    def close(self) -> None:
        """Unmap the neighbours' buffers and free this rank's (after a device
        sync and a barrier-free contract: call it on every rank once no rank
        will send any more)."""
        torch.cuda.synchronize(self.device)
        for pb in self._peers:
            pb.close()
        self._peers = []
        for b in (self._flags_buf, *self._rings):
            if b is not None:
                b.free()

    def check(self) -> None:
        """Raise if a transfer timed out (syncs)."""
        if int(self.status.item()) != 0:
            raise RuntimeError(f"stage {self.rank}: peer transfer timed out (a neighbour never signalled)")


def _capture_debugger():
    """PO_DEBUG_CAPTURE=1: report the first op after which the current
    stream's capture became invalidated (diagnostics only)."""
    import os

    if os.environ.get("PO_DEBUG_CAPTURE") != "1":
        return None
    import ctypes
    import sys

    cudart = ctypes.CDLL("libcudart.so.12")
    st = ctypes.c_int()
    seen = [False]

    def probe(where):
        cudart.cudaStreamIsCapturing(ctypes.c_void_p(torch.cuda.current_stream().cuda_stream), ctypes.byref(st))
        if st.value == 2 and not seen[0]:
            seen[0] = True
            print(f"[peer] capture invalidated by {where}", file=sys.stderr, flush=True)

    return probe


def _stream(device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


class PeerStageRunner:
    """Runs one stage's 1F1B program on this rank over peer-memory rings;
    `capture()` turns one full run into a CUDA graph that `replay()` re-runs
    (continuing training: optimizer scalars come from a CoefTape refreshed
    before each replay). Data must be device-resident; checks are deferred."""

    def __init__(self, dist, tl: Timeline, stage, opt, strategy: str, data, loss_kind: str, lr_for_mb, rows: int,
                 *, fuse: bool = True, group=None, stage_ranks: list[int] | None = None, timeout_ms: int = 60_000,
                 dp_rank: int = 0, dp_size: int = 1, fused_dp=None):
        """Hybrid DP x PP: stage_ranks[k] is the global rank of stage k in this
        replica; replica `dp_rank` of `dp_size` trains on rows [dp_rank*rows,
        (dp_rank+1)*rows) of every batch, and `fused_dp` (a
        dp_fused.FusedDPGroup over the stage's replicas) folds the gradient
        mean into the update (device epochs, so the run stays one graph)."""
        if STRATEGY_SCHEDULE.get(strategy) != "1f1b" or tl.kind != "1f1b":
            raise ValueError(f"the peer runner executes 1f1b strategies, got {strategy!r} on {tl.kind!r}")
        if strategy == "spectrain" and opt.config.kind != "sgdm":
            raise ValueError("spectrain requires the sgdm optimizer")
        validate_timeline(tl)
        self.tl, self.stage, self.opt, self.strategy = tl, stage, opt, strategy
        self.rank, self.depth = stage.rank, tl.depth
        self.data, self.loss_kind, self.lr_for_mb, self.rows, self.fuse = data, loss_kind, lr_for_mb, rows, fuse
        self.device = stage.flat.device
        self.predictive = strategy in PREDICTIVE_STRATEGIES
        self.program = stage_program(tl, self.rank, predictive=self.predictive)
        slots = ring_slots(tl)
        self.links = PeerLinks(dist, self.rank, self.depth, rows, stage.in_shape, stage.out_shape, slots,
                               self.device, group=group, stage_ranks=stage_ranks, timeout_ms=timeout_ms)
        opt.eager_checks = False
        self.graph = None
        self.runs = 0
        self._pending = None
        if (dp_size > 1) != (fused_dp is not None):
            raise ValueError("data parallelism (dp_size > 1) needs a fused_dp group, and only then")
        self.dp_rank, self.dp_size, self.fused_dp = dp_rank, dp_size, fused_dp
        self._scratch = None
        if fused_dp is not None:
            stage.set_grad_buffer(fused_dp.grad)

    def _issue(self, lr_fn):
        """Enqueue one full run of this rank's program on the current stream."""
        st, links, last = self.stage, self.links, self.rank == self.depth - 1
        policy = _make_policy(self.strategy, self.tl)
        rt = _StageRt(st, self.opt, self.depth)
        if self.fused_dp is not None:
            self.fused_dp.adopt(st, self.opt, rt)  # shard mode: peer-mapped W, state, W_hat
        else:  # W_hat in the gradient's storage (runtime._StageRt)
            rt.alias_grad = staging_in_grad_ok(st, policy.predictive, self.tl.micro_per_mini)
        st.version = 1
        work = [op for op in self.program if op.kind != UPDATE]
        flags = torch.ones(len(work), dtype=torch.bool, device=self.device)
        losses = torch.zeros(self.tl.n_batches, dtype=torch.float32, device=self.device) if last else None
        records: dict[int, VersionRecord] = {}
        order: list[VersionRecord] = []
        local_grads: dict[int, torch.Tensor] = {}
        snapshot_peak, wi = 1, 0
        debug = _capture_debugger()
        for op in self.program:
            if debug is not None:
                debug(f"rank {self.rank} before {op.kind}{op.mb}")
            if op.kind == UPDATE:
                lr = lr_fn(op.mb)
                fuse = self.fuse and op.fuse_predict
                if self.fused_dp is not None:  # replicas' gradient mean inside K3
                    if fuse:
                        out, lr_p, gap = rt.staging_buffer(), lr_fn(op.next_mb), op.next_gap
                    elif self.fused_dp.mode == "shard":  # a plain step: no prediction output
                        out, lr_p, gap = None, 0.0, 0
                    else:  # a plain step: the prediction output goes to scratch
                        if self._scratch is None:
                            self._scratch = st.flat.layout.empty(self.device)
                        out, lr_p, gap = self._scratch, 0.0, 0
                    self.fused_dp.step_predict_dev(self.opt, st.flat, lr, lr_p, gap, out)
                    st.set_grad_buffer(self.fused_dp.grad)
                elif fuse:
                    self.opt.step_predict_(st.flat, lr, lr_fn(op.next_mb), op.next_gap, rt.staging_buffer())
                else:
                    self.opt.step_(st.flat, lr)
                if fuse:
                    rt.prepared = (op.next_mb, op.next_gap)
                st.version += 1
                rt.pending_count = 0
                policy.after_update(rt)
            elif op.kind == FORWARD:
                x = links.recv_act() if self.rank > 0 else self._shard(_to_device(self.data.batch(op.mb)[0],
                                                                                    self.device))
                weights, fv, predicted, target = policy.forward_view(rt, op.mb, 0, lr_fn(op.mb))
                if last:  # forward + loss (+ dL/dout) in one launch for a narrow output layer
                    y = self._shard(_to_device(self.data.batch(op.mb)[1], self.device))
                    out, loss, grad = st.run_forward_loss(weights, (op.mb, 0), x, fv, y, self.loss_kind,
                                                          check_finite=False, finite_flags=flags, flag_index=wi)
                else:
                    out = st.run_forward(weights, (op.mb, 0), x, fv, check_finite=False, finite_flags=flags,
                                         flag_index=wi)
                rec = VersionRecord(op.mb, 0, self.rank, fv, predicted, target)
                records[op.mb] = rec
                order.append(rec)
                if last:
                    losses[op.mb - 1] = loss
                    local_grads[op.mb] = grad
                else:
                    links.send_act(out if out.is_contiguous() else out.contiguous())
                wi += 1
            else:
                g_out = local_grads.pop(op.mb) if last else links.recv_grad()
                rec = records[op.mb]
                weights, bv = policy.backward_view(rt, op.mb, 0, rec.forward_version)
                g_in, _ = st.run_backward(weights, (op.mb, 0), g_out, accumulate=False, need_input_grad=self.rank > 0)
                rt.pending_count = 1
                rec.backward_version = bv
                rec.live_backward_version = st.version
                if self.rank > 0:
                    links.send_grad(g_in if g_in.is_contiguous() else g_in.contiguous())
                wi += 1
            snapshot_peak = max(snapshot_peak, policy.snapshot_count(rt))
        return order, flags, losses, snapshot_peak, work

    def _shard(self, t):
        if self.dp_size == 1:
            return t
        return t[self.dp_rank * self.rows : (self.dp_rank + 1) * self.rows]

    def run(self) -> StageReport:
        """One eager run (asynchronous device work, one sync at the end)."""
        t0 = time.perf_counter()
        self._pending = self._issue(self.lr_for_mb)
        self.runs += 1
        return self.report(time.perf_counter() - t0)

    def capture(self) -> None:
        """Capture one full run into a CUDA graph (run() at least once first:
        it warms cuBLAS/cuDNN and the optimizer state)."""
        if self.runs == 0:
            raise RuntimeError("run() once before capture()")
        if self.fused_dp is not None and self.tl.n_batches % 2:
            raise ValueError("a captured DP run must hold an even number of updates (grad-buffer parity)")
        self.opt._ensure_state()
        torch.cuda.synchronize(self.device)
        self.tape = CoefTape(self.device)
        base = self.opt.step_count
        self.graph = torch.cuda.CUDAGraph()
        self.tape.begin([self.opt])
        try:
            with capture(self.graph):
                self._pending = self._issue(lambda mb: MbLr(self.lr_for_mb(mb), mb))
        finally:
            self.tape.end([self.opt])
        self.updates = self.opt.step_count - base
        self.opt.step_count = base  # nothing ran during capture
        self.launches = len(self.tape.entries)

    def replay(self) -> None:
        """Enqueue one more full run (asynchronous)."""
        self.tape.refresh({id(self.opt): self.opt.step_count}, self.lr_for_mb)
        self.graph.replay()
        self.opt.step_count += self.updates
        self.stage.version = self.tl.n_batches + 1
        self.runs += 1

    def report(self, seconds: float = 0.0) -> StageReport:
        """StageReport of the most recent run (synchronises; raises on a
        transfer timeout or a non-finite forward output / loss / update)."""
        order, flags, losses, snapshot_peak, work = self._pending
        self.links.check()
        if self.fused_dp is not None:
            self.fused_dp.check()
        if not bool(flags.all()):
            bad = int((~flags).nonzero()[0].item())
            raise NumericError(f"mb {work[bad].mb} stage {self.rank}: non-finite value in stage forward output")
        self.opt.check_finite()
        host_losses = None
        if losses is not None:
            host_losses = losses.cpu().tolist()
            if not all(v == v and abs(v) != float("inf") for v in host_losses):
                raise NumericError(f"stage {self.rank}: non-finite loss under {self.loss_kind}")
        if self.stage.version != self.tl.n_batches + 1 or len(self.stage.stash):
            raise RuntimeError(f"stage {self.rank} did not drain: version {self.stage.version}")
        executed = [(op.kind, op.mb) for op in self.program]
        return StageReport(self.rank, order, host_losses, self.stage.version, self.stage.stash.peak, snapshot_peak,
                           seconds, executed)


__all__ = ["PeerLinks", "PeerStageRunner", "ring_slots"]


# ---- bench support ---------------------------------------------------------------------------


_BENCH_BROKEN: list = []  # a failed peer leg disables the later ones (each would wait out its timeouts)


def bench_peer_pipeline(torch_mod, dist, rank, world, device, make_stage, data, loss_kind, lr, rows, n_batches,
                        replays: int = 5, trials: int = 3, opt_kind: str = "adam", opt_kw: dict | None = None,
                        timeout_ms: int = 15_000):
    """Prediction off/on through the peer runner, one CUDA graph per rank per
    run: eager warm-up run, capture, one warm replay, then `trials` x
    `replays` timed replays per arm in alternation (median; device time of
    the replays, max over ranks). `make_stage()` -> this rank's stage."""
    import statistics

    from .optim import OptimizerConfig, OptimizerState
    from .runtime import build_timeline

    if _BENCH_BROKEN:
        raise RuntimeError(f"skipped: an earlier peer leg failed ({_BENCH_BROKEN[0]})")
    runners = {}
    try:
        for strategy in ("async_raw", "optimizer_prediction"):
            stage = make_stage()
            opt = OptimizerState(OptimizerConfig(opt_kind, **(opt_kw or {})), stage.param_names, device=device)
            r = PeerStageRunner(dist, build_timeline(strategy, world, n_batches), stage, opt, strategy, data,
                                loss_kind, lambda mb: lr, rows, timeout_ms=timeout_ms)
            r.run()
            r.capture()
            r.replay()
            r.report()
            runners[strategy] = r
    except Exception as exc:
        _BENCH_BROKEN.append(f"{type(exc).__name__}: {exc}")
        raise
    times = {s: [] for s in runners}
    for _ in range(trials):
        for s, r in runners.items():
            torch_mod.cuda.synchronize(device)
            dist.barrier()
            e0, e1 = torch_mod.cuda.Event(enable_timing=True), torch_mod.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(replays):
                r.replay()
            e1.record()
            torch_mod.cuda.synchronize(device)
            t = torch_mod.tensor([e0.elapsed_time(e1) / 1e3 / replays], device=device)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            times[s].append(float(t.item()))
    out = {}
    for s, r in runners.items():
        r.report()  # raises on a transfer timeout or a non-finite value
        key = "pred_on" if s == "optimizer_prediction" else "pred_off"
        sec = statistics.median(times[s])
        out[key] = {"samples_per_s": round(n_batches * rows / sec, 1), "s_per_run": round(sec, 5),
                    "s_per_run_trials": [round(t, 5) for t in times[s]], "graph_launches_per_run": r.launches}
    out["prediction_overhead"] = round(1.0 - out["pred_on"]["samples_per_s"] / out["pred_off"]["samples_per_s"], 4)
    torch_mod.cuda.synchronize(device)
    dist.barrier()  # no rank sends any more: free the rings
    for r in runners.values():
        r.graph = None
        r.links.close()
    runners.clear()
    torch_mod.cuda.empty_cache()
    return out
