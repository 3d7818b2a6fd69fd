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
)
from .schedule import BACKWARD, FORWARD, UPDATE, Timeline, stage_program, validate_timeline
from .stages import StageModel, loss_and_grad


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


class _StagedRecv:
    """Completion handle of a host-staged receive: wait(), then copy to device."""

    def __init__(self, reqs, host, dev):
        self.reqs, self.host, self.dev = reqs, host, dev

    def wait(self):
        for r in self.reqs:
            r.wait()
        self.dev.copy_(self.host)

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
        reqs = d.batch_isend_irecv(ops)
        self.inflight.append((reqs, [t for t, _ in sends]))
        if self.host_staging and staged:
            return [_StagedRecv(reqs, staged[0][0], staged[0][1])]
        return reqs

    def drain(self):
        for reqs, _ in self.inflight:
            for r in reqs:
                r.wait()
        self.inflight.clear()


class PipelineStageRunner:
    """Runs one stage's 1F1B program on this rank."""

    def __init__(self, dist, tl: Timeline, stage: StageModel, opt, strategy: str, data, loss_kind: str,
                 lr_for_mb, rows: int, *, checks: str = "deferred", fuse: bool = True, group=None,
                 stage_ranks: list[int] | None = None, dp_group=None, dp_rank: int = 0, dp_size: int = 1,
                 host_staging: bool = False, fused_dp=None):
        """stage_ranks[k] is the global rank holding stage k of this pipeline
        replica (default: rank k). With dp_size > 1 (hybrid DP x PP), replica
        `dp_rank` trains on rows [dp_rank*rows, (dp_rank+1)*rows) of every
        batch and the stage gradient is averaged over `dp_group` before each
        update, so the replicas stay identical."""
        if STRATEGY_SCHEDULE.get(strategy) != "1f1b" or tl.kind != "1f1b":
            raise ValueError(f"the distributed runner executes 1f1b strategies, got {strategy!r} on {tl.kind!r}")
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
            self._scratch = None
        opt.eager_checks = self.eager

    # -- what each op consumes / produces -------------------------------------------------

    def _input_spec(self, op):
        if op.kind == FORWARD and self.rank > 0:
            return (self.rows, *self.stage.in_shape), self.stage_ranks[self.rank - 1]
        if op.kind == BACKWARD and self.rank < self.depth - 1:
            return (self.rows, *self.stage.out_shape), self.stage_ranks[self.rank + 1]
        return None

    def run(self) -> StageReport:
        work = [op for op in self.program if op.kind != UPDATE]
        records: dict[int, VersionRecord] = {}
        order: list[VersionRecord] = []
        losses = {} if self.rank == self.depth - 1 else None
        grads_local: dict[int, torch.Tensor] = {}
        snapshot_peak = 1
        executed = []
        flags = torch.ones(len(work), dtype=torch.bool, device=self.device)
        t0 = time.perf_counter()

        def post_recv(op):
            spec = self._input_spec(op)
            if spec is None:
                return None, []
            buf = torch.empty(spec[0], dtype=torch.float32, device=self.device)
            return buf, [(buf, spec[1])]

        nxt_buf, recv = post_recv(work[0]) if work else (None, [])
        nxt_req = self.comm.post([], recv)
        wi = 0
        i = 0
        while i < len(self.program):
            op = self.program[i]
            i += 1
            executed.append((op.kind, op.mb))
            if op.kind == UPDATE:
                self._update(op)
                snapshot_peak = max(snapshot_peak, self.policy.snapshot_count(self.rt))
                continue
            inp, req = nxt_buf, nxt_req
            for r in req:
                r.wait()
            out_msg = None
            if op.kind == FORWARD:
                if self.rank == 0:
                    inp = self._shard(_to_device(self.data.batch(op.mb)[0], self.device))
                weights, fv, predicted, target = self.policy.forward_view(self.rt, op.mb, 0, self.lr_for_mb(op.mb))
                try:
                    out = self.stage.run_forward(weights, (op.mb, 0), inp, fv, check_finite=self.eager,
                                                 finite_flags=flags, flag_index=wi)
                except NumericError as err:
                    raise NumericError(f"mb {op.mb} stage {self.rank}: {err}") from err
                rec = VersionRecord(op.mb, 0, self.rank, fv, predicted, target)
                records[op.mb] = rec
                order.append(rec)
                if self.rank < self.depth - 1:
                    out_msg = (out.contiguous(), self.stage_ranks[self.rank + 1])
                else:
                    y = self._shard(_to_device(self.data.batch(op.mb)[1], self.device))
                    loss, g = loss_and_grad(out, y, self.loss_kind)
                    if self.eager and not bool(torch.isfinite(loss)):
                        raise NumericError(f"mb {op.mb} stage {self.rank}: non-finite loss under {self.loss_kind}")
                    losses[op.mb] = loss.detach()
                    grads_local[op.mb] = g
            else:
                g_out = grads_local.pop(op.mb) if self.rank == self.depth - 1 else inp
                rec = records[op.mb]
                weights, bv = self.policy.backward_view(self.rt, op.mb, 0, rec.forward_version)
                g_in, _ = self.stage.run_backward(weights, (op.mb, 0), g_out, accumulate=False,
                                                  need_input_grad=self.rank > 0)
                self.rt.pending_count = 1
                rec.backward_version = bv
                rec.live_backward_version = self.stage.version
                if self.rank > 0:
                    out_msg = (g_in.contiguous(), self.stage_ranks[self.rank - 1])
            snapshot_peak = max(snapshot_peak, self.policy.snapshot_count(self.rt))
            wi += 1
            # one grouped exchange: this op's output + the next work op's input
            if wi < len(work):
                nxt_buf, recv = post_recv(work[wi])
            else:
                nxt_buf, recv = None, []
            nxt_req = self.comm.post([out_msg] if out_msg else [], recv)
        self.comm.drain()
        if self.fused_dp is not None:
            self.fused_dp.check()
        if not self.eager:
            if not bool(flags.all()):
                bad = int((~flags).nonzero()[0].item())
                raise NumericError(f"mb {work[bad].mb} stage {self.rank}: non-finite value in stage forward output")
            self.opt.check_finite()
        host_losses = None
        if losses is not None:
            vals = torch.stack([losses[m] for m in sorted(losses)]).cpu().tolist()
            host_losses = vals
            if not all(v == v and abs(v) != float("inf") for v in vals):
                raise NumericError(f"stage {self.rank}: non-finite loss under {self.loss_kind}")
        if self.stage.version != self.tl.n_batches + 1 or len(self.stage.stash):
            raise RuntimeError(f"stage {self.rank} did not drain: version {self.stage.version}")
        return StageReport(self.rank, order, host_losses, self.stage.version, self.stage.stash.peak,
                           snapshot_peak, time.perf_counter() - t0, executed)

    def _shard(self, t):
        if self.dp_size == 1:
            return t
        return t[self.dp_rank * self.rows : (self.dp_rank + 1) * self.rows]

    def _update(self, op):
        if self.fused_dp is not None:
            lr = self.lr_for_mb(op.mb)
            if self.fuse and op.fuse_predict:
                out, lr_p, gap = self.rt.staging_buffer(), self.lr_for_mb(op.next_mb), op.next_gap
                self.rt.prepared = (op.next_mb, op.next_gap)
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
    for strategy in ("async_raw", "optimizer_prediction"):
        times = []
        for trial in range(2):  # trial 0 warms NCCL / cuBLAS
            group = partition_layers(layers, world)[rank]
            stage = StageModel(rank, group, torch_init(0, device), device)
            opt = OptimizerState(OptimizerConfig("adam"), stage.param_names, device=device)
            tl = build_timeline(strategy, world, n_batches if trial else 2 * world + 2)
            runner = PipelineStageRunner(dist, tl, stage, opt, strategy, data, "softmax_xent", lambda mb: 1e-4,
                                         BATCH, host_staging=host_staging)
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
        out[key] = {"samples_per_s": round(n_batches * BATCH / float(t.item()), 1), "s": round(float(t.item()), 4)}
    on, off = out["pred_on"]["samples_per_s"], out["pred_off"]["samples_per_s"]
    out.update(value=on, unit="samples/s", prediction_overhead=round(1.0 - on / off, 4),
               launches=n_batches * 2)
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
    torch_mod.backends.cuda.matmul.allow_tf32 = False
    torch_mod.backends.cudnn.allow_tf32 = False
    return out


def bench_hybrid_dp_pp(torch_mod, dist, rank, world, device, n_batches: int = 32, host_staging: bool = False):
    """DP 2 x PP world/2 on config-1-shaped stages (each replica half of every
    B = 128 batch): the stage-gradient mean by NCCL all-reduce + K3 vs the
    fused peer-memory mean inside K3 (dp_fused). Samples/s, max over ranks."""
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
    for arm in ("nccl_allreduce", "fused_peer_mean"):
        times = []
        for trial, n in enumerate((2 * pp + 2, n_batches)):
            stage = StageModel(k, partition_layers(layers, pp)[k], torch_init(0, device), device)
            opt = OptimizerState(OptimizerConfig("adam"), stage.param_names, device=device)
            fused = (FusedDPGroup(dist, groups[k], r, dp, stage.flat.layout.numel, device)
                     if arm == "fused_peer_mean" else None)
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
        t = torch_mod.tensor([times[-1]], device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        out[arm] = {"samples_per_s": round(n_batches * BATCH / float(t.item()), 1), "s": round(float(t.item()), 4)}
    return out
