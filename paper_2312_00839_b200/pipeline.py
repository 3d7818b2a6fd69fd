"""One-process-per-GPU 1F1B pipeline runner (NCCL point-to-point over NVLink).

Each rank owns stage `rank` of a depth-`world` pipeline and executes its own
program — `stage_program(tl, rank)`, i.e. exactly the reference's
`tl.stage_events(rank)` order (pkg/src/pipesim/schedule.py:80-81), which the
reference simulates in one thread (runtime.py:404-466) — with the same
weight policies, version bookkeeping and kernels as the single-process
runner (runtime.py in this package).

Communication: activations flow rank k -> k+1 after forwards, input
gradients k+1 -> k after backwards. After every work op the rank posts ONE
grouped exchange {send its output, receive the next op's input}
(torch.distributed.batch_isend_irecv -> ncclGroupStart/End). In 1F1B the two
neighbours' groups pair up exactly ({send a_m, recv g_j} on k matches
{send g_j, recv a_m} on k+1), which is what makes the schedule deadlock-free
on a single communicator, and the transfers run on NCCL's stream while the
compute stream runs the UPDATE (K2/K3) that follows every backward.
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import torch

from .errors import NumericError
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
from .stages import StageModel


@dataclass
class StageReport:
    rank: int
    records: list
    losses: list | None
    final_version: int
    stash_peak: int
    snapshot_peak: int
    seconds: float
    executed: list


def input_link(kind, stage: int, depth: int):
    """The boundary message a work op of `stage` consumes: ("act", k) is the
    activation k -> k+1, ("grad", k) the input gradient k+1 -> k; None for
    stage 0's forwards and the last stage's backwards (local inputs)."""
    if kind == FORWARD and stage > 0:
        return ("act", stage - 1)
    if kind == BACKWARD and stage < depth - 1:
        return ("grad", stage)
    return None


def output_link(kind, stage: int, depth: int):
    """The boundary message a work op of `stage` produces (None: kept local)."""
    if kind == FORWARD and stage < depth - 1:
        return ("act", stage)
    if kind == BACKWARD and stage > 0:
        return ("grad", stage - 1)
    return None


def exchange_plan(program, stage: int, depth: int) -> list[list[tuple[str, tuple, int]]]:
    """The grouped exchanges PipelineStageRunner.run posts, in posting order:
    group 0 = {recv work[0]'s input}; group i+1 = {send work[i]'s output,
    recv work[i+1]'s input} — entries ("send" | "recv", link, (mb, micro)). Every group
    is one batch_isend_irecv (ncclGroupStart/End); tests/test_nccl_groups.py
    checks that these plans cannot deadlock under NCCL's group semantics."""
    work = [op for op in program if op.kind != UPDATE]
    groups = []
    first = input_link(work[0].kind, stage, depth) if work else None
    groups.append([("recv", first, (work[0].mb, work[0].micro))] if first else [])
    for i, op in enumerate(work):
        g = []
        out = output_link(op.kind, stage, depth)
        if out:
            g.append(("send", out, (op.mb, op.micro)))
        if i + 1 < len(work):
            nxt = input_link(work[i + 1].kind, stage, depth)
            if nxt:
                g.append(("recv", nxt, (work[i + 1].mb, work[i + 1].micro)))
        groups.append(g)
    return groups


class _Req:
    """A communication request whose wait() may be called more than once: a
    gloo send's wait consumes its completion, so a second wait (the run loop
    waits every posted request before the next op; the graphed runner waits a
    slot's previous send again before overwriting its buffer) would block."""

    __slots__ = ("work", "done")

    def __init__(self, work):
        self.work, self.done = work, False

    def wait(self):
        if not self.done:
            self.work.wait()
            self.done = True

    def is_completed(self):
        return self.done or self.work.is_completed()


class _StagedRecv:
    """Completion handle of a host-staged receive: wait(), then copy to device."""

    def __init__(self, reqs, host, dev):
        self.reqs, self.host, self.dev = reqs, host, dev
        self.done = False

    def wait(self):
        if self.done:  # idempotent: a second wait must not re-copy stale data
            return
        for r in self.reqs:
            r.wait()
        self.dev.copy_(self.host)
        self.done = True

    def is_completed(self):
        return all(r.is_completed() for r in self.reqs)


class _Exchange:
    """Grouped neighbour P2P for one rank.

    host_staging=True moves device tensors through host memory (for a
    backend without device transport, e.g. gloo with several ranks on one
    GPU in the tests); with NCCL the device buffers go over NVLink directly.
    """

    def __init__(self, dist, group=None, host_staging: bool = False):
        self.dist = dist
        self.group = group
        self.host_staging = host_staging
        self.inflight: list = []  # (request, tensor) kept alive until complete

    def post(self, sends, recvs):
        """sends: [(tensor, peer)], recvs: [(buffer, peer)] -> requests for recvs."""
        d = self.dist
        self.inflight = [(rq, ts) for rq, ts in self.inflight if not all(r.is_completed() for r in rq)]
        if self.host_staging:
            sends = [(t.cpu(), peer) for t, peer in sends]
            staged = [(torch.empty(b.shape, dtype=b.dtype), b, peer) for b, peer in recvs]
            recvs = [(h, peer) for h, _, peer in staged]
        ops = [d.P2POp(d.isend, t, peer, self.group) for t, peer in sends]
        ops += [d.P2POp(d.irecv, b, peer, self.group) for b, peer in recvs]
        if not ops:
            return []
        reqs = [_Req(w) for w in d.batch_isend_irecv(ops)]
        self.inflight.append((reqs, [t for t, _ in sends]))
        if self.host_staging and staged:
            return [_StagedRecv(reqs, staged[0][0], staged[0][1])]
        return reqs

    def drain(self):
        for reqs, _ in self.inflight:
            for r in reqs:
                r.wait()
        self.inflight.clear()


class _SlotTape:
    """A one-slot coefficient tape: graph-captured optimizer launches read
    their scalars from one device po_coef that is refilled (host double
    arithmetic, po_coef_fill) before each replay. The pinned staging is a ring
    so the host never overwrites a slot whose H2D copy may still be pending."""

    RING = 8

    def __init__(self, device):
        from . import _lib

        self._lib = _lib
        self.dev = torch.zeros(4, dtype=torch.float32, device=device)
        self.host = torch.zeros(self.RING * 4, dtype=torch.float32).pin_memory()
        self.done = [None] * self.RING
        self.k = 0

    def record(self, opt, which, lr, lr_pred, steps_ahead):
        return self.dev.data_ptr()

    def fill(self, opt, which, lr, lr_times_s):
        import ctypes

        k = self.k
        self.k = (k + 1) % self.RING
        if self.done[k] is not None:
            self.done[k].synchronize()
        host = self.host[4 * k : 4 * k + 4]
        rc = self._lib.load().po_coef_fill(ctypes.byref(opt._hp), which, float(lr), float(lr_times_s),
                                           opt.step_count, host.data_ptr())
        self._lib.check(rc, "po_coef_fill")
        self.dev.copy_(host, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        self.done[k] = ev


class _OpGraphs:
    """Per-(op kind, stash slot) CUDA graphs of one rank's stage work.

    The first occurrence of an op in a slot runs eagerly (it also warms
    cuBLAS on the stream), the second is captured and replayed, later ones
    replay. Every cross-op tensor lives at a static address: receive buffers
    per slot, the forward's stash / output / loss per slot (graph pool), the
    live and staging weights, the flat gradient. Slots are mb mod D (at most
    D - k mini-batches are in flight on stage k). Optimizer updates replay a
    K2 or K3 graph whose scalars come from a _SlotTape refilled on the host
    before each replay.
    """

    def __init__(self, runner: "PipelineStageRunner"):
        self.r = runner
        self.slots = runner.depth
        self.count: dict = {}
        self.graphs: dict = {}
        self.recv: dict = {}
        self.xbuf: dict = {}
        self.ybuf: dict = {}
        self.sends: dict = {}
        self.tape = _SlotTape(runner.device)

    def _slot(self, mb):
        return mb % self.slots

    def recv_buffer(self, op, shape):
        key = (op.kind, self._slot(op.mb))
        buf = self.recv.get(key)
        if buf is None or tuple(buf.shape) != tuple(shape):
            buf = self.recv[key] = torch.empty(shape, dtype=torch.float32, device=self.r.device)
        return buf

    def _static(self, table, slot, t):
        buf = table.get(slot)
        if buf is None or buf.shape != t.shape:
            buf = table[slot] = torch.empty_like(t)
        buf.copy_(t)
        return buf

    def _run(self, key, fn):
        """Eager on the first occurrence, capture + replay on the second,
        replay afterwards. Returns fn's outputs (graph-owned when captured)."""
        n = self.count.get(key, 0)
        self.count[key] = n + 1
        if n == 0:
            return fn()
        if n == 1:
            graph = torch.cuda.CUDAGraph()
            with capture(graph):
                outs = fn()
            self.graphs[key] = (graph, outs)
        graph, outs = self.graphs[key]
        graph.replay()
        return outs

    def _wait_send(self, key):
        for w in self.sends.pop(key, []):
            w.wait()

    def sent(self, op, reqs):
        self.sends[(op.kind, self._slot(op.mb))] = list(reqs)

    def forward(self, op, weights, x, y, fv, flags, flag_base):
        r, slot = self.r, self._slot(op.mb)
        st = r.stage
        self._wait_send((op.kind, slot))  # the slot's previous output must have left
        if r.rank == 0:
            x = self._static(self.xbuf, slot, x)
        if y is not None:
            y = self._static(self.ybuf, slot, y)
        last = r.rank == r.depth - 1

        def fn():
            if last:
                return st.run_forward_loss(weights, ("slot", slot), x, fv, y, r.loss_kind, check_finite=False,
                                           finite_flags=flags, flag_index=flag_base + slot)
            out = st.run_forward(weights, ("slot", slot), x, fv, check_finite=False, finite_flags=flags,
                                 flag_index=flag_base + slot)
            return out, None, None

        return self._run(("F", slot, weights[0].data_ptr()), fn)

    def backward(self, op, weights, g_out):
        r, slot = self.r, self._slot(op.mb)
        self._wait_send((op.kind, slot))

        def fn():
            g_in, _ = r.stage.run_backward(weights, ("slot", slot), g_out, accumulate=False,
                                           need_input_grad=r.rank > 0)
            return g_in

        # keyed on the weights' address like the forward: under weight stashing
        # / 2BW the backward reads a per-version snapshot whose address the
        # captured graph bakes in
        return self._run(("B", slot, weights[0].data_ptr()), fn)

    def update(self, op):
        from . import _lib

        r = self.r
        lr = r.lr_for_mb(op.mb)
        fused = r.fuse and op.fuse_predict
        key = ("U", fused)
        first = self.count.get(key, 0) == 0
        if fused:
            lr_p, gap = r.lr_for_mb(op.next_mb), op.next_gap
            r.rt.staging_buffer()

            def fn():
                r.opt.step_predict_(r.stage.flat, lr, lr_p, gap, r.rt.staging)

            which, c = _lib.PO_COEF_STEP_PREDICT, float(lr_p) * gap
        else:

            def fn():
                r.opt.step_(r.stage.flat, lr)

            which, c = _lib.PO_COEF_STEP, 0.0
        if first:
            fn()  # eager (advances step_count itself)
            self.count[key] = 1
        else:
            if self.count[key] == 1:  # capture with the slot tape; nothing runs during capture
                r.opt._ensure_state()
                sc = r.opt.step_count
                r.opt.tape = self.tape
                graph = torch.cuda.CUDAGraph()
                try:
                    with capture(graph):
                        fn()
                finally:
                    r.opt.tape = None
                    r.opt.step_count = sc
                self.graphs[key] = (graph, None)
                self.count[key] = 2
            self.tape.fill(r.opt, which, lr, c)
            self.graphs[key][0].replay()
            r.opt.step_count += 1
        if fused:
            r.rt.prepared = (op.next_mb, op.next_gap)
        r.stage.version += 1
        r.rt.pending_count = 0
        r.policy.after_update(r.rt)


class PipelineStageRunner:
    """Runs one stage's 1F1B (or GPipe) program on this rank."""

    def __init__(self, dist, tl: Timeline, stage: StageModel, opt, strategy: str, data, loss_kind: str,
                 lr_for_mb, rows: int, *, checks: str = "deferred", fuse: bool = True, group=None,
                 stage_ranks: list[int] | None = None, dp_group=None, dp_rank: int = 0, dp_size: int = 1,
                 host_staging: bool = False, fused_dp=None, graphed: bool = False):
        """stage_ranks[k] is the global rank holding stage k of this pipeline
        replica (default: rank k). With dp_size > 1 (hybrid DP x PP), replica
        `dp_rank` trains on rows [dp_rank*rows, (dp_rank+1)*rows) of every
        batch and the stage gradient is averaged over `dp_group` before each
        update, so the replicas stay identical."""
        kind = STRATEGY_SCHEDULE.get(strategy)
        if kind not in ("1f1b", "gpipe") or tl.kind != kind:
            raise ValueError(f"the distributed runner executes 1f1b and gpipe strategies, got {strategy!r} "
                             f"on {tl.kind!r}")
        if rows % tl.micro_per_mini:
            raise ValueError(f"{rows} rows do not split into {tl.micro_per_mini} micro-batches")
        if strategy == "spectrain" and opt.config.kind != "sgdm":
            raise ValueError("spectrain requires the sgdm optimizer")
        validate_timeline(tl)
        self.dist = dist
        self.tl = tl
        self.stage = stage
        self.opt = opt
        self.rank = stage.rank
        self.depth = tl.depth
        self.strategy = strategy
        self.data = data
        self.loss_kind = loss_kind
        self.lr_for_mb = lr_for_mb
        self.rows = rows
        # GPipe: T micro-batches of rows / T per mini-batch, gradients summed
        # over them and averaged before the update (runtime.py:441-454)
        self.micros = tl.micro_per_mini
        self.mrows = rows // self.micros
        self.eager = checks == "eager"
        self.fuse = fuse
        self.predictive = strategy in PREDICTIVE_STRATEGIES
        self.policy = _make_policy(strategy, tl)
        self.rt = _StageRt(stage, opt, self.depth)
        self.program = stage_program(tl, self.rank, predictive=self.predictive)
        self.comm = _Exchange(dist, group, host_staging=host_staging)
        self.device = stage.flat.device
        self.stage_ranks = stage_ranks or list(range(self.depth))
        self.dp_group, self.dp_rank, self.dp_size = dp_group, dp_rank, dp_size
        # fused_dp: a dp_fused.FusedDPGroup — the DP mean is read from the
        # replicas' peer-mapped gradients inside the K3 pass (no all-reduce)
        self.fused_dp = fused_dp
        if fused_dp is not None:
            stage.set_grad_buffer(fused_dp.grad)
            fused_dp.adopt(stage, opt, self.rt)  # shard mode: peer-mapped W, state, W_hat
            self._scratch = None
        else:  # W_hat in the gradient's storage (runtime._StageRt)
            self.rt.alias_grad = staging_in_grad_ok(stage, self.predictive, self.micros)
        opt.eager_checks = self.eager
        # graphed=True: every op's device work is captured once per (kind,
        # stash slot) into a CUDA graph and replayed (the eager per-op Python
        # cost dominates small stages); needs deferred checks, an MLP stage
        # and no data parallelism (those paths run eagerly)
        use_graphs = (graphed and not self.eager and dp_size == 1 and isinstance(stage, StageModel)
                      and self.device.type == "cuda" and self.micros == 1)
        self._graphs = _OpGraphs(self) if use_graphs else None

    # -- what each op consumes / produces -------------------------------------------------

    def _input_spec(self, op):
        link = input_link(op.kind, self.rank, self.depth)
        if link is None:
            return None
        if link[0] == "act":
            return (self.mrows, *self.stage.in_shape), self.stage_ranks[self.rank - 1]
        return (self.mrows, *self.stage.out_shape), self.stage_ranks[self.rank + 1]

    def run(self) -> StageReport:
        work = [op for op in self.program if op.kind != UPDATE]
        records: dict[int, VersionRecord] = {}
        order: list[VersionRecord] = []
        losses = {} if self.rank == self.depth - 1 else None
        grads_local: dict[tuple[int, int], torch.Tensor] = {}
        snapshot_peak = 1
        executed = []
        g = self._graphs
        # finiteness flags: one per eager forward (by work index), one per
        # graphed slot (po_all_finite only ever clears a flag)
        flags = torch.ones(len(work) + (g.slots if g else 0), dtype=torch.bool, device=self.device)
        in_flight = peak_in_flight = 0
        t0 = time.perf_counter()

        def post_recv(op):
            spec = self._input_spec(op)
            if spec is None:
                return None, []
            buf = g.recv_buffer(op, spec[0]) if g else torch.empty(spec[0], dtype=torch.float32, device=self.device)
            return buf, [(buf, spec[1])]

        nxt_buf, recv = post_recv(work[0]) if work else (None, [])
        nxt_req = self.comm.post([], recv)
        wi = 0
        i = 0
        while i < len(self.program):
            op = self.program[i]
            i += 1
            executed.append((op.kind, op.mb) if self.micros == 1 else (op.kind, op.mb, op.micro))
            if op.kind == UPDATE:
                if g is not None:
                    g.update(op)
                else:
                    self._update(op)
                snapshot_peak = max(snapshot_peak, self.policy.snapshot_count(self.rt))
                continue
            inp, req = nxt_buf, nxt_req
            for r in req:
                r.wait()
            out_msg = None
            if op.kind == FORWARD:
                x = inp
                y = None
                last = self.rank == self.depth - 1
                if self.rank == 0:
                    x = self._micro(self._shard(_to_device(self.data.batch(op.mb)[0], self.device)), op.micro)
                if last:
                    y = self._micro(self._shard(_to_device(self.data.batch(op.mb)[1], self.device)), op.micro)
                weights, fv, predicted, target = self.policy.forward_view(self.rt, op.mb, op.micro,
                                                                          self.lr_for_mb(op.mb))
                try:
                    if g is not None:
                        out, loss, grad = g.forward(op, weights, x, y, fv, flags, len(work))
                    else:
                        if last:
                            out, loss, grad = self.stage.run_forward_loss(
                                weights, (op.mb, op.micro), x, fv, y, self.loss_kind, check_finite=self.eager,
                                finite_flags=flags, flag_index=wi)
                        else:
                            out = self.stage.run_forward(weights, (op.mb, op.micro), x, fv,
                                                         check_finite=self.eager, finite_flags=flags, flag_index=wi)
                            loss = grad = None
                except NumericError as err:
                    raise NumericError(f"mb {op.mb} stage {self.rank}: {err}") from err
                in_flight += 1
                peak_in_flight = max(peak_in_flight, in_flight)
                rec = VersionRecord(op.mb, op.micro, self.rank, fv, predicted, target)
                records[(op.mb, op.micro)] = rec
                order.append(rec)
                if output_link(op.kind, self.rank, self.depth):
                    out_msg = (out if out.is_contiguous() else out.contiguous(), self.stage_ranks[self.rank + 1])
                else:
                    if self.eager and not bool(torch.isfinite(loss)):
                        raise NumericError(f"mb {op.mb} stage {self.rank}: non-finite loss under {self.loss_kind}")
                    losses.setdefault(op.mb, []).append(loss.detach().clone() if g is not None else loss.detach())
                    grads_local[(op.mb, op.micro)] = grad
            else:
                g_out = grads_local.pop((op.mb, op.micro)) if self.rank == self.depth - 1 else inp
                rec = records[(op.mb, op.micro)]
                weights, bv = self.policy.backward_view(self.rt, op.mb, op.micro, rec.forward_version)
                if g is not None:
                    g_in = g.backward(op, weights, g_out)
                else:
                    g_in, _ = self.stage.run_backward(weights, (op.mb, op.micro), g_out,
                                                      accumulate=self.rt.pending_count > 0,
                                                      need_input_grad=self.rank > 0)
                in_flight -= 1
                self.rt.pending_count += 1
                rec.backward_version = bv
                rec.live_backward_version = self.stage.version
                if output_link(op.kind, self.rank, self.depth):
                    out_msg = (g_in if g_in.is_contiguous() else g_in.contiguous(), self.stage_ranks[self.rank - 1])
            snapshot_peak = max(snapshot_peak, self.policy.snapshot_count(self.rt))
            wi += 1
            # one grouped exchange: this op's output + the next work op's input
            if wi < len(work):
                nxt_buf, recv = post_recv(work[wi])
            else:
                nxt_buf, recv = None, []
            nxt_req = self.comm.post([out_msg] if out_msg else [], recv)
            if g is not None and out_msg is not None:
                g.sent(op, nxt_req)
        self.comm.drain()
        if self.fused_dp is not None:
            self.fused_dp.check()
        if not self.eager:
            if not bool(flags.all()):
                bad = int((~flags).nonzero()[0].item())
                where = f"mb {work[bad].mb}" if bad < len(work) else f"mb slot {bad - len(work)} (graphed)"
                raise NumericError(f"{where} stage {self.rank}: non-finite value in stage forward output")
            self.opt.check_finite()
        host_losses = None
        if losses is not None:
            vals = torch.stack([torch.stack(losses[m]).mean() if len(losses[m]) > 1 else losses[m][0]
                                for m in sorted(losses)]).cpu().tolist()
            host_losses = vals
            if not all(v == v and abs(v) != float("inf") for v in vals):
                raise NumericError(f"stage {self.rank}: non-finite loss under {self.loss_kind}")
        if self.stage.version != self.tl.n_batches + 1 or len(self.stage.stash):
            raise RuntimeError(f"stage {self.rank} did not drain: version {self.stage.version}")
        stash_peak = max(self.stage.stash.peak, peak_in_flight)
        return StageReport(self.rank, order, host_losses, self.stage.version, stash_peak,
                           snapshot_peak, time.perf_counter() - t0, executed)

    def _micro(self, t, micro: int):
        if self.micros == 1:
            return t
        return t[micro * self.mrows : (micro + 1) * self.mrows]

    def _shard(self, t):
        if self.dp_size == 1:
            return t
        return t[self.dp_rank * self.rows : (self.dp_rank + 1) * self.rows]

    def _update(self, op):
        if self.rt.pending_count > 1:  # GPipe: mean over the micro-batches (runtime.py:441-454)
            self.stage.flat.grad.div_(self.rt.pending_count)
        if self.fused_dp is not None:
            lr = self.lr_for_mb(op.mb)
            if self.fuse and op.fuse_predict:
                out, lr_p, gap = self.rt.staging_buffer(), self.lr_for_mb(op.next_mb), op.next_gap
                self.rt.prepared = (op.next_mb, op.next_gap)
            elif self.fused_dp.mode == "shard":  # plain step: no prediction output
                out, lr_p, gap = None, 0.0, 0
            else:  # plain step: the prediction output goes to scratch
                if self._scratch is None:
                    self._scratch = self.stage.flat.layout.empty(self.device)
                out, lr_p, gap = self._scratch, 0.0, 0
            self.fused_dp.step_predict(self.opt, self.stage.flat, lr, lr_p, gap, out)
            if self.eager:
                self.opt.check_finite()
                self.fused_dp.check()
            self.stage.set_grad_buffer(self.fused_dp.grad)
            self.stage.version += 1
            self.rt.pending_count = 0
            self.policy.after_update(self.rt)
            return
        if self.dp_size > 1:
            # hybrid DP x PP: mean gradient over the data-parallel replicas of
            # this stage, then the (fused) update on identical replicas
            self.dist.all_reduce(self.stage.flat.grad, group=self.dp_group)
            self.stage.flat.grad.mul_(1.0 / self.dp_size)
        lr = self.lr_for_mb(op.mb)
        try:
            if self.fuse and op.fuse_predict:
                self.opt.step_predict_(self.stage.flat, lr, self.lr_for_mb(op.next_mb), op.next_gap,
                                       self.rt.staging_buffer())
                self.rt.prepared = (op.next_mb, op.next_gap)
            else:
                self.opt.step_(self.stage.flat, lr)
        except NumericError as err:
            raise NumericError(f"mb {op.mb} stage {self.rank}: {err}") from err
        self.stage.version += 1
        self.rt.pending_count = 0
        self.policy.after_update(self.rt)


def gather_reports(dist, report: StageReport, world: int):
    """All stage reports on every rank (object all-gather)."""
    out = [None] * world
    dist.all_gather_object(out, report)
    return out


# ---- bench support ---------------------------------------------------------------------------


def bench_config1_pipeline(torch_mod, dist, rank, world, device, n_batches: int = 64, host_staging: bool = False):
    """Config-1-shaped pipeline on `world` GPUs: prediction on vs off, samples/s
    (device-timed per rank, max over ranks)."""
    from .bench_pipeline import BATCH, CONFIG1_ACTS, CONFIG1_DIMS, DeviceBatches
    from .optim import OptimizerConfig, OptimizerState
    from .runtime import build_timeline
    from .stages import build_layers, partition_layers, torch_init

    torch_mod.backends.cuda.matmul.allow_tf32 = False
    if world <= 4:
        dims, acts = CONFIG1_DIMS, CONFIG1_ACTS
    else:  # config 1 has 4 layers; one more 1024-wide ReLU layer per extra stage
        dims = [3072] + [1024] * (world - 1) + [10]
        acts = ["relu"] * (world - 1) + ["linear"]
    layers = build_layers(dims, acts)
    data = DeviceBatches(torch_mod, device, dims=dims)
    out = {"config": f"MLP {dims}, B={BATCH}, Adam lr 1e-4, 1F1B D={world} (one stage per GPU, NCCL P2P), "
                     f"{n_batches} mini-batches, fp32 GEMMs"}
    for graphed in (False, True):
        for strategy in ("async_raw", "optimizer_prediction"):
            times = []
            for trial in range(2):  # trial 0 warms NCCL / cuBLAS
                group = partition_layers(layers, world)[rank]
                stage = StageModel(rank, group, torch_init(0, device), device)
                opt = OptimizerState(OptimizerConfig("adam"), stage.param_names, device=device)
                tl = build_timeline(strategy, world, n_batches if trial else 2 * world + 2)
                runner = PipelineStageRunner(dist, tl, stage, opt, strategy, data, "softmax_xent", lambda mb: 1e-4,
                                             BATCH, host_staging=host_staging, graphed=graphed)
                torch_mod.cuda.synchronize(device)
                dist.barrier()
                e0, e1 = torch_mod.cuda.Event(enable_timing=True), torch_mod.cuda.Event(enable_timing=True)
                e0.record()
                runner.run()
                e1.record()
                torch_mod.cuda.synchronize(device)
                dist.barrier()
                times.append(e0.elapsed_time(e1) / 1e3)
            t = torch_mod.tensor([times[-1]], device=device)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            key = ("graphed_" if graphed else "") + ("pred_on" if strategy == "optimizer_prediction" else "pred_off")
            out[key] = {"samples_per_s": round(n_batches * BATCH / float(t.item()), 1),
                        "s": round(float(t.item()), 4)}
    on, off = out["pred_on"]["samples_per_s"], out["pred_off"]["samples_per_s"]
    gon, goff = out["graphed_pred_on"]["samples_per_s"], out["graphed_pred_off"]["samples_per_s"]
    out.update(value=max(on, gon), unit="samples/s", prediction_overhead=round(1.0 - on / off, 4),
               graphed_prediction_overhead=round(1.0 - gon / goff, 4), launches=n_batches * 2)
    # GPipe on the same stages and GPUs (T = 4 micro-batches, eager NCCL runner)
    try:
        times = []
        for trial in range(2):
            stage = StageModel(rank, partition_layers(layers, world)[rank], torch_init(0, device), device)
            opt = OptimizerState(OptimizerConfig("adam"), stage.param_names, device=device)
            nb = n_batches if trial else 2
            tl = build_timeline("gpipe", world, nb, 4)
            runner = PipelineStageRunner(dist, tl, stage, opt, "gpipe", data, "softmax_xent", lambda mb: 1e-4, BATCH,
                                         host_staging=host_staging)
            torch_mod.cuda.synchronize(device)
            dist.barrier()
            e0, e1 = torch_mod.cuda.Event(enable_timing=True), torch_mod.cuda.Event(enable_timing=True)
            e0.record()
            runner.run()
            e1.record()
            torch_mod.cuda.synchronize(device)
            dist.barrier()
            times.append(e0.elapsed_time(e1) / 1e3)
        t = torch_mod.tensor([times[-1]], device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        out["gpipe_t4"] = {"samples_per_s": round(n_batches * BATCH / float(t.item()), 1), "s": round(float(t.item()), 4)}
        out["pipeoptim_over_gpipe"] = round(on / out["gpipe_t4"]["samples_per_s"], 4)
    except Exception as exc:
        out["gpipe_t4"] = {"error": f"rank {rank}: {type(exc).__name__}: {exc}"}
    # counted-work bound for one stage per GPU (roofline.py)
    from .roofline import mlp_pipeline_bounds
    from .stages import build_stages

    cpu_stages = build_stages(layers, world, torch_init(0, torch_mod.device("cpu")), device="cpu")
    bound = mlp_pipeline_bounds(cpu_stages, BATCH, n_batches, "adam", True, "fast_fp32")
    out["roofline"] = {"one_stage_per_gpu": bound["one_stage_per_gpu"], "per_stage": bound["per_stage"],
                       "peak_source": bound["peak_source"]}
    # the peer-memory transport: a rank's whole run is one CUDA graph (no NCCL,
    # no host in the loop); reported beside the NCCL runner and, when faster,
    # as the value
    try:
        from .peer_pipeline import bench_peer_pipeline

        peer = bench_peer_pipeline(
            torch_mod, dist, rank, world, device,
            lambda: StageModel(rank, partition_layers(layers, world)[rank], torch_init(0, device), device),
            data, "softmax_xent", 1e-4, BATCH, n_batches)
        out["peer_graphed"] = peer
        if peer["pred_on"]["samples_per_s"] > out["value"]:
            out.update(value=peer["pred_on"]["samples_per_s"], transport="peer memory (one CUDA graph per rank)",
                       prediction_overhead=peer["prediction_overhead"])
    except Exception as exc:  # the NCCL numbers above still stand
        import sys
        import traceback

        traceback.print_exc(file=sys.stderr)
        out["peer_graphed"] = {"error": f"rank {rank}: {type(exc).__name__}: {exc}"}
    out["frac_of_roofline"] = round(out["value"] / bound["one_stage_per_gpu"]["samples_per_s"], 4)
    return out


def bench_module_pipeline(torch_mod, dist, rank, world, device, name: str, n_batches: int = 16,
                          host_staging: bool = False):
    """Configs 2-4 on `world` GPUs, one stage per GPU (depth = world):
    prediction on vs off, samples/s device-timed, max over ranks."""
    from .bench_pipeline import MODULE_CONFIGS, ModuleBatches, module_block_costs, module_stages_for
    from .optim import OptimizerConfig, OptimizerState
    from .runtime import build_timeline

    cfg = MODULE_CONFIGS[name]
    # one partition for every rank: rank 0's profiled costs, broadcast
    box = [module_block_costs(torch_mod, name, device) if rank == 0 else None]
    dist.broadcast_object_list(box, src=0)
    costs = box[0]
    torch_mod.backends.cuda.matmul.allow_tf32 = True
    torch_mod.backends.cudnn.allow_tf32 = True
    data = ModuleBatches(torch_mod, device, cfg)
    out = {"config": f"{name}: D={world} (one stage per GPU, NCCL P2P), batch {cfg['batch']}, {cfg['opt']}, "
                     f"{n_batches} mini-batches, TF32 convs/GEMMs, fp32 master weights"}
    for strategy in ("async_raw", "optimizer_prediction"):
        times = []
        for trial, n in enumerate((2 * world, n_batches)):
            stages, _ = module_stages_for(torch_mod, name, device, depth=world, costs=costs)
            stage = stages[rank]
            for k, st in enumerate(stages):  # only this rank's stage stays on the device
                if k != rank:
                    st.module.to("cpu")
            del stages
            kw = {"weight_decay": 5e-4} if cfg["opt"] == "sgdm" else {}
            opt = OptimizerState(OptimizerConfig(cfg["opt"], **kw), stage.param_names, device=device)
            tl = build_timeline(strategy, world, n)
            runner = PipelineStageRunner(dist, tl, stage, opt, strategy, data, "softmax_xent", lambda mb: cfg["lr"],
                                         cfg["batch"], host_staging=host_staging)
            torch_mod.cuda.synchronize(device)
            dist.barrier()
            e0, e1 = torch_mod.cuda.Event(enable_timing=True), torch_mod.cuda.Event(enable_timing=True)
            e0.record()
            runner.run()
            e1.record()
            torch_mod.cuda.synchronize(device)
            dist.barrier()
            times.append(e0.elapsed_time(e1) / 1e3)
        t = torch_mod.tensor([times[-1]], device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        key = "pred_on" if strategy == "optimizer_prediction" else "pred_off"
        out[key] = {"samples_per_s": round(n_batches * cfg["batch"] / float(t.item()), 2), "s": round(float(t.item()), 4)}
    on, off = out["pred_on"]["samples_per_s"], out["pred_off"]["samples_per_s"]
    out.update(value=on, unit="samples/s", prediction_overhead=round(1.0 - on / off, 4))
    try:  # the peer-memory transport, one CUDA graph per rank per run
        from .peer_pipeline import bench_peer_pipeline

        def make_stage():
            from .stage_models import use_cudnn_bn

            stages, _ = module_stages_for(torch_mod, name, device, depth=world, costs=costs)
            for k, st in enumerate(stages):
                if k != rank:
                    st.module.to("cpu")
            # the peer runner keeps all of a rank's work on one stream (its waits
            # included): cuDNN's grid-synchronising batch norm is safe there
            use_cudnn_bn([stages[rank]])
            return stages[rank]

        kw = {"weight_decay": 5e-4} if cfg["opt"] == "sgdm" else {}
        peer = bench_peer_pipeline(torch_mod, dist, rank, world, device, make_stage, data, "softmax_xent",
                                   cfg["lr"], cfg["batch"], n_batches, replays=2, trials=3, opt_kind=cfg["opt"],
                                   opt_kw=kw)
        out["peer_graphed"] = peer
        if peer["pred_on"]["samples_per_s"] > out["value"]:
            out.update(value=peer["pred_on"]["samples_per_s"], transport="peer memory (one CUDA graph per rank)",
                       prediction_overhead=peer["prediction_overhead"])
    except Exception as exc:
        import sys
        import traceback

        traceback.print_exc(file=sys.stderr)
        out["peer_graphed"] = {"error": f"rank {rank}: {type(exc).__name__}: {exc}"}
    torch_mod.backends.cuda.matmul.allow_tf32 = False
    torch_mod.backends.cudnn.allow_tf32 = False
    return out


def bench_hybrid_dp_pp(torch_mod, dist, rank, world, device, n_batches: int = 32, host_staging: bool = False):
    """DP 2 x PP world/2 on config-1-shaped stages (each replica half of every
    B = 128 batch): the stage-gradient mean by NCCL all-reduce + K3 vs the
    fused peer-memory mean inside K3 (dp_fused, every replica reading every
    gradient) vs the sharded form (reduce-scatter + K3 + all-gather in one
    pass). Samples/s, max over ranks."""
    from .bench_pipeline import BATCH, CONFIG1_ACTS, CONFIG1_DIMS, DeviceBatches
    from .dp_fused import FusedDPGroup
    from .optim import OptimizerConfig, OptimizerState
    from .runtime import build_timeline
    from .stages import build_layers, partition_layers, torch_init

    dp, pp = 2, world // 2
    if world % 2 or pp < 1:
        return {"error": f"hybrid leg needs an even world size, got {world}"}
    torch_mod.backends.cuda.matmul.allow_tf32 = False
    r, k = divmod(rank, pp)
    groups = [dist.new_group([q * pp + s for q in range(dp)]) for s in range(pp)]
    if pp <= 4:
        dims, acts = CONFIG1_DIMS, CONFIG1_ACTS
    else:
        dims, acts = [3072] + [1024] * (pp - 1) + [10], ["relu"] * (pp - 1) + ["linear"]
    layers = build_layers(dims, acts)
    data = DeviceBatches(torch_mod, device, dims=dims)
    out = {"config": f"DP {dp} x PP {pp}, MLP {dims}, B={BATCH} ({BATCH // dp} rows per replica), Adam, "
                     f"optimizer_prediction, {n_batches} mini-batches"}
    for arm in ("nccl_allreduce", "fused_peer_mean", "fused_shard"):
        times = []
        for trial, n in enumerate((2 * pp + 2, n_batches)):
            stage = StageModel(k, partition_layers(layers, pp)[k], torch_init(0, device), device)
            opt = OptimizerState(OptimizerConfig("adam"), stage.param_names, device=device)
            fused = (FusedDPGroup(dist, groups[k], r, dp, stage.flat.layout.numel, device,
                                  mode="shard" if arm == "fused_shard" else "peer_load")
                     if arm != "nccl_allreduce" else None)
            runner = PipelineStageRunner(dist, build_timeline("optimizer_prediction", pp, n), stage, opt,
                                         "optimizer_prediction", data, "softmax_xent", lambda mb: 1e-4, BATCH // dp,
                                         stage_ranks=[r * pp + s for s in range(pp)], dp_group=groups[k],
                                         dp_rank=r, dp_size=dp, fused_dp=fused, host_staging=host_staging)
            torch_mod.cuda.synchronize(device)
            dist.barrier()
            e0, e1 = torch_mod.cuda.Event(enable_timing=True), torch_mod.cuda.Event(enable_timing=True)
            e0.record()
            runner.run()
            e1.record()
            torch_mod.cuda.synchronize(device)
            dist.barrier()
            times.append(e0.elapsed_time(e1) / 1e3)
            if fused is not None:
                fused.close(dist, groups[k])
        t = torch_mod.tensor([times[-1]], device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        out[arm] = {"samples_per_s": round(n_batches * BATCH / float(t.item()), 1), "s": round(float(t.item()), 4)}
    # the same hybrid on the peer runner: neighbour rings + the fused DP mean on
    # device epochs, a rank's whole run as one CUDA graph
    try:
        from .peer_pipeline import PeerStageRunner

        stage = StageModel(k, partition_layers(layers, pp)[k], torch_init(0, device), device)
        opt = OptimizerState(OptimizerConfig("adam"), stage.param_names, device=device)
        fused = FusedDPGroup(dist, groups[k], r, dp, stage.flat.layout.numel, device, timeout_ms=15_000)
        runner = PeerStageRunner(dist, build_timeline("optimizer_prediction", pp, n_batches), stage, opt,
                                 "optimizer_prediction", data, "softmax_xent", lambda mb: 1e-4, BATCH // dp,
                                 stage_ranks=[r * pp + s for s in range(pp)], dp_rank=r, dp_size=dp, fused_dp=fused,
                                 timeout_ms=15_000)
        runner.run()
        runner.capture()
        runner.replay()
        runner.report()
        torch_mod.cuda.synchronize(device)
        dist.barrier()
        e0, e1 = torch_mod.cuda.Event(enable_timing=True), torch_mod.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            runner.replay()
        e1.record()
        torch_mod.cuda.synchronize(device)
        runner.report()
        t = torch_mod.tensor([e0.elapsed_time(e1) / 1e3 / 3], device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        out["peer_graphed_fused_mean"] = {"samples_per_s": round(n_batches * BATCH / float(t.item()), 1),
                                          "s": round(float(t.item()), 4)}
        dist.barrier()
        runner.links.close()
    except Exception as exc:
        out["peer_graphed_fused_mean"] = {"error": f"rank {rank}: {type(exc).__name__}: {exc}"}
    return out
