"""Hybrid DP x PP with the data-parallel gradient reduction fused into the
optimizer pass ("the grad allreduce fused ahead of K3").

The replicas of one pipeline stage map each other's flat gradient buffers
(CUDA IPC; over NVLink / NVSwitch on a multi-GPU node) and each runs ONE
kernel, `po_step_predict_dp`, that reads the dp gradients of every element
from peer memory, sums them in rank order (identical on every replica, so
replicas stay bit-identical), and applies the fused step + prediction (K3).
Compared with NCCL all-reduce followed by K3 this saves the reduced
gradient's HBM write and re-read and one launch, and overlaps the NVLink
reads with the local HBM stream.

Synchronisation: after its backward a replica release-stores the epoch into
every replica's flag array (`po_dp_signal`); the fused kernel's CTAs
acquire-wait on their local flags. Gradients are double-buffered by epoch
parity (see csrc/pipeoptim_kernels.cu for why that needs no second
handshake). The kernel times out (status flag) instead of hanging if a
replica never signals.

`mode="shard"` (po_step_predict_dp_shard) is the reduce-scatter + K3 +
all-gather form: the replicas' weights, optimizer state and W_hat staging
buffer live in peer-mapped memory too, replica r computes only its 1/dp
shard (gradient sum over the peers, K3 against its own W / state) and stores
the results into every replica's buffers; a done-barrier then makes the
whole update visible before the next forward. Per GPU that moves
~(20 + 12/dp) B/param through HBM instead of (28 + 4 dp), and
~20 (dp-1)/dp B/param per NVLink direction instead of 4 (dp-1): the
peer-load form wins at small dp, the sharded one from dp ~ 4.
The same kernel reads the gradient through multimem.ld_reduce and writes
through multimem.st when the buffers are bound to NVLS multicast objects
(`po_dp_multicast`); on this round's one-GPU boxes cuMulticastCreate is
refused (profiles/r2_nvls_probe.txt), so only the peer-store transport runs.
"""

from __future__ import annotations

import ctypes
import os
import socket

import torch

from . import _lib


def send_fd(dist, group, rank: int, size: int, fd, error: str | None = None):
    """Pass a file descriptor from replica 0 to replicas 1..size-1 of `group`
    over an abstract UNIX socket (SCM_RIGHTS); returns the received fd on the
    others (a new descriptor the caller owns), None on replica 0. Used for
    the NVLS multicast object's POSIX handle. Replica 0 passes `error`
    instead of a descriptor when it could not make one: every replica then
    raises it (nobody is left waiting on the socket)."""
    token = [(os.urandom(8).hex(), error) if rank == 0 else None]
    dist.broadcast_object_list(token, src=_group_src(dist, group), group=group)
    tok, err = token[0]
    if err is not None:
        raise RuntimeError(f"replica 0 could not share the handle: {err}")
    name = f"\0pipeoptim-fd-{os.getuid()}-{tok}"
    if rank == 0:
        with socket.socket(socket.AF_UNIX, socket.SOCK_STREAM) as srv:
            srv.bind(name)
            srv.listen(size)
            dist.barrier(group=group)
            for _ in range(size - 1):
                conn, _ = srv.accept()
                with conn:
                    socket.send_fds(conn, [b"fd"], [fd])
        dist.barrier(group=group)
        return None
    dist.barrier(group=group)
    with socket.socket(socket.AF_UNIX, socket.SOCK_STREAM) as c:
        c.connect(name)
        _, fds, _, _ = socket.recv_fds(c, 16, 1)
    dist.barrier(group=group)
    return fds[0]


def _group_src(dist, group) -> int:
    """Global rank of the group's replica 0 (broadcast_object_list takes a
    global source rank)."""
    if group is None:
        return 0
    return dist.get_global_rank(group, 0)


class FusedDPGroup:
    """Peer-mapped, double-buffered gradients of one stage's DP replicas
    (shard mode: also the weights, optimizer state and W_hat)."""

    MODES = ("peer_load", "shard")
    TRANSPORTS = ("peer", "nvls")
    _BIG = ("grad0", "grad1", "w", "s1", "s2", "w_hat")  # fp32 [numel] each

    def __init__(self, dist, group, dp_rank: int, dp_size: int, numel: int, device, timeout_ms: int = 60_000,
                 mode: str = "peer_load", transport: str = "peer"):
        from .ipc import IpcBuffer, open_peer

        if not 1 <= dp_size <= 8:
            raise ValueError(f"fused DP supports 1..8 replicas, got {dp_size}")
        if mode not in self.MODES:
            raise ValueError(f"fused DP mode must be one of {self.MODES}, got {mode!r}")
        if transport not in self.TRANSPORTS or (transport == "nvls" and mode != "shard"):
            raise ValueError(f"transport must be 'peer', or 'nvls' with mode='shard'; got {transport!r}")
        self.dp_rank, self.dp_size, self.numel, self.mode, self.transport = dp_rank, dp_size, numel, mode, transport
        self.device = torch.device(device)
        self.timeout_ms = timeout_ms
        self._lib = _lib.load()
        big = self._BIG if mode == "shard" else self._BIG[:2]
        # node-shared (CUDA IPC) buffers, mapped by each peer into its own
        # device (ipc.py): the big fp32 buffers (unless NVLS-bound) and the
        # flag arrays (gradient-ready [dp], done [dp], non-finite [1])
        ipc_specs = [] if transport == "nvls" else [(name, numel, torch.float32) for name in big]
        ipc_specs.append(("flags", dp_size, torch.int64))
        if mode == "shard":
            ipc_specs += [("done", dp_size, torch.int64), ("bad", 1, torch.int64)]
        self._ipc = {name: IpcBuffer(n, dt, self.device) for name, n, dt in ipc_specs}
        self.local = {name: b.tensor for name, b in self._ipc.items()}
        self.mc = None  # per gradient parity: po_dp_multicast (NVLS transport)
        self._nvls = None
        if transport == "nvls":
            self._bind_nvls(dist, group, big)
        if "bad" in self.local:
            self.local["bad"].fill_(2 ** 63 - 1)
        self.bufs = [self.local["grad0"], self.local["grad1"]]
        self.flags = self.local["flags"]
        self.status = torch.zeros(1, dtype=torch.int32, device=self.device)
        self.poisoned = False
        self.closed = False
        torch.cuda.synchronize(self.device)
        names = list(self._ipc)
        mine = [self._ipc[n].export() for n in names]
        handles = [None] * dp_size
        dist.all_gather_object(handles, mine, group=group)
        self._opened = []
        # peer[name][r]: replica r's buffer mapped here (own buffers for r == dp_rank,
        # and for every r where the transport is NVLS — those are reached via multicast)
        self.peer = {n: [None] * dp_size for n in self.local}
        for r, h in enumerate(handles):
            for n, x in zip(names, h):
                if r == dp_rank:
                    self.peer[n][r] = self.local[n]
                else:
                    pb = open_peer(x, self.device)
                    self._opened.append(pb)
                    self.peer[n][r] = pb.tensor
        for n in self.local:
            if n not in self._ipc:
                self.peer[n] = [self.local[n]] * dp_size
        # slot of THIS replica in every replica's flag array
        self.slots = torch.tensor([t.data_ptr() + 8 * dp_rank for t in self.peer["flags"]], dtype=torch.int64,
                                  device=self.device)
        P = ctypes.c_void_p * dp_size
        col = lambda n: P(*[t.data_ptr() for t in self.peer[n]])  # noqa: E731
        self.grad_ptrs = [col("grad0"), col("grad1")]
        self.epoch = 0
        self.parity = 0
        if mode == "shard":
            self.w_ptrs, self.s1_ptrs, self.s2_ptrs, self.what_ptrs = col("w"), col("s1"), col("s2"), col("w_hat")
            self.bad_ptrs = col("bad")
            self.done = self.local["done"]
            # slot of THIS replica in every replica's done array (device array)
            self.done_slots = torch.tensor([t.data_ptr() + 8 * dp_rank for t in self.peer["done"]],
                                           dtype=torch.int64, device=self.device)
            lo, hi = ctypes.c_int64(), ctypes.c_int64()
            _lib.check(self._lib.po_dp_shard_range(numel, dp_size, dp_rank, ctypes.byref(lo), ctypes.byref(hi)),
                       "po_dp_shard_range")
            self.shard = (lo.value, hi.value)
            self._adopted = False
        # CUDA-graph form (step_predict_dev): the epoch lives on the device
        self.epoch_ctr = torch.zeros(1, dtype=torch.int64, device=self.device)
        self._slot = None
        dist.barrier(group=group)

    def _bind_nvls(self, dist, group, big) -> None:
        """One NVLS multicast object over all the replicas' big buffers:
        replica 0 creates it and passes its POSIX fd to the others over a
        UNIX socket (SCM_RIGHTS); every replica adds its device, then binds its
        own physical memory and maps the unicast and multicast addresses."""
        from .ipc import _wrap

        region = self.numel * 4
        total = region * len(big)
        lib = self._lib
        h = ctypes.c_void_p()
        if self.dp_rank == 0:
            fd = ctypes.c_int32(-1)
            rc = lib.po_nvls_create(self.dp_size, total, ctypes.byref(fd), ctypes.byref(h))
            if rc != 0:  # tell the other replicas before raising (they wait in send_fd)
                err = f"po_nvls_create: {lib.po_strerror(rc).decode()} (rc {rc})"
                send_fd(dist, group, self.dp_rank, self.dp_size, None, error=err)
            send_fd(dist, group, self.dp_rank, self.dp_size, fd.value)
            os.close(fd.value)
            rc = 0
        else:
            fd = send_fd(dist, group, self.dp_rank, self.dp_size, None)
            rc = lib.po_nvls_open(fd, self.dp_size, total, ctypes.byref(h))
            os.close(fd)
        if rc == 0:
            self._nvls = h
            rc = lib.po_nvls_add_device(h)
        self._agree(dist, group, rc, "po_nvls_open / po_nvls_add_device")  # every device is in the team ...
        uc, mc = ctypes.c_void_p(), ctypes.c_void_p()
        rc = lib.po_nvls_bind(h, ctypes.byref(uc), ctypes.byref(mc))  # ... before anyone binds
        self._agree(dist, group, rc, "po_nvls_bind")
        for i, name in enumerate(big):
            self.local[name] = _wrap(uc.value + i * region, self.numel, torch.float32, self.device)
        at = {name: mc.value + i * region for i, name in enumerate(big)}
        self.mc = [_lib.po_dp_multicast(at[g], at["w"], at["s1"], at["s2"], at["w_hat"]) for g in ("grad0", "grad1")]

    def _agree(self, dist, group, rc: int, what: str) -> None:
        """A collective step: every replica learns whether all succeeded, so
        a failure raises everywhere instead of leaving peers in a barrier."""
        codes = [None] * self.dp_size
        dist.all_gather_object(codes, int(rc), group=group)
        bad = [(r, c) for r, c in enumerate(codes) if c != 0]
        if bad:
            r, c = bad[0]
            raise RuntimeError(f"{what} failed on replica {r}: {self._lib.po_strerror(c).decode()} (rc {c})")

    @property
    def grad(self) -> torch.Tensor:
        """The buffer this replica's next backward must write into."""
        return self.bufs[self.parity]

    def adopt(self, stage, opt, rt=None) -> None:
        """Shard mode: move the stage's live weights, the optimizer state and
        non-finite flag, and the W_hat staging buffer (rt: runtime._StageRt)
        into the peer-mapped buffers the owners write into (once), and point
        `rt`'s staging buffer at the peer-mapped W_hat (every run's _StageRt).
        A no-op in peer_load mode."""
        if self.mode != "shard":
            return
        lay = stage.flat.layout
        if lay.numel != self.numel:
            raise ValueError("stage size does not match the DP group's buffers")
        if rt is not None:
            rt.staging = self.local["w_hat"]
            rt.staging_views = lay.views(rt.staging)
        if self._adopted:
            return
        opt._bind(lay)
        opt._ensure_state()
        stage.set_weight_buffer(self.local["w"])
        self.local["s1"].copy_(opt._s1)
        opt._s1 = self.local["s1"]
        if opt._s2 is not None:
            self.local["s2"].copy_(opt._s2)
            opt._s2 = self.local["s2"]
        self.local["bad"].copy_(opt._bad)
        opt._bad = self.local["bad"]
        self._adopted = True

    @property
    def staging(self) -> torch.Tensor | None:
        """Shard mode: the peer-mapped W_hat buffer (the stage's staging buffer)."""
        return self.local["w_hat"] if self.mode == "shard" else None

    def _shard_call(self, opt, flat, out, lr, c_pred, step_count, coef, epoch, epoch_dev, stream) -> None:
        if not self._adopted or flat.data.data_ptr() != self.local["w"].data_ptr():
            raise RuntimeError("sharded DP: adopt(stage, opt, rt) must move the stage's buffers first")
        if out is not None and out.data_ptr() != self.local["w_hat"].data_ptr():
            raise ValueError("sharded DP: the prediction output must be the group's peer-mapped staging buffer")
        mc = ctypes.byref(self.mc[self.parity]) if self.mc is not None else None
        rc = self._lib.po_step_predict_dp_shard(
            ctypes.byref(opt._hp), self.dp_size, self.dp_rank, self.w_ptrs, self.grad_ptrs[self.parity],
            self.s1_ptrs, None if opt._s2 is None else self.s2_ptrs, None if out is None else self.what_ptrs,
            self.numel, float(lr), float(c_pred), step_count, coef, self.bad_ptrs, self.flags.data_ptr(),
            self.done_slots.data_ptr(), self.done.data_ptr(), epoch, epoch_dev, self.timeout_ms,
            self.status.data_ptr(), mc, stream)
        _lib.check(rc, "po_step_predict_dp_shard")

    def step_predict(self, opt, flat, lr: float, lr_pred: float, steps_ahead: int, out: torch.Tensor) -> None:
        """Signal this epoch's gradient, then the fused mean-over-replicas K3."""
        self._live()
        if steps_ahead < 0:
            raise ValueError(f"steps_ahead must be >= 0, got {steps_ahead}")
        if flat.layout.numel != self.numel:
            raise ValueError("stage size does not match the DP group's buffers")
        opt._bind(flat.layout)
        opt._ensure_state()
        self.epoch += 1
        stream = torch.cuda.current_stream(self.device).cuda_stream
        _lib.check(self._lib.po_dp_signal(self.slots.data_ptr(), self.dp_size, self.epoch, stream), "po_dp_signal")
        if self.mode == "shard":
            self._shard_call(opt, flat, out, lr, float(lr_pred) * steps_ahead, opt.step_count, None, self.epoch, None,
                             stream)
            opt.step_count += 1
            self.parity ^= 1
            return
        rc = self._lib.po_step_predict_dp(
            ctypes.byref(opt._hp), flat.data.data_ptr(), self.grad_ptrs[self.parity], self.dp_size,
            opt._s1.data_ptr(), None if opt._s2 is None else opt._s2.data_ptr(), out.data_ptr(), self.numel,
            float(lr), float(lr_pred) * steps_ahead, opt.step_count, opt._bad.data_ptr(), self.flags.data_ptr(),
            self.epoch, self.timeout_ms, self.status.data_ptr(), stream,
        )
        _lib.check(rc, "po_step_predict_dp")
        opt.step_count += 1
        self.parity ^= 1

    def step_predict_dev(self, opt, flat, lr, lr_pred, steps_ahead: int, out: torch.Tensor) -> None:
        """step_predict for CUDA-graph capture and replay: the epoch is a device
        counter (po_dp_signal_dev / po_step_predict_dp_dc) and the step's
        scalars come from the optimizer's CoefTape while capturing (else from
        a device po_coef filled here). The grad-buffer parity alternates per
        call as in step_predict, so a captured run must hold an even number
        of updates to replay consistently."""
        self._live()
        if steps_ahead < 0:
            raise ValueError(f"steps_ahead must be >= 0, got {steps_ahead}")
        if flat.layout.numel != self.numel:
            raise ValueError("stage size does not match the DP group's buffers")
        opt._bind(flat.layout)
        opt._ensure_state()
        stream = torch.cuda.current_stream(self.device).cuda_stream
        _lib.check(self._lib.po_dp_signal_dev(self.slots.data_ptr(), self.dp_size, self.epoch_ctr.data_ptr(), stream),
                   "po_dp_signal_dev")
        if opt.tape is not None:
            coef = opt.tape.record(opt, _lib.PO_COEF_STEP_PREDICT, lr, lr_pred, steps_ahead)
        else:
            if self._slot is None:
                from .pipeline import _SlotTape

                self._slot = _SlotTape(self.device)
            self._slot.fill(opt, _lib.PO_COEF_STEP_PREDICT, lr, float(lr_pred) * steps_ahead)
            coef = self._slot.dev.data_ptr()
        if self.mode == "shard":
            self._shard_call(opt, flat, out, 0.0, 0.0, 0, coef, 0, self.epoch_ctr.data_ptr(), stream)
            opt.step_count += 1
            self.parity ^= 1
            return
        rc = self._lib.po_step_predict_dp_dc(
            ctypes.byref(opt._hp), flat.data.data_ptr(), self.grad_ptrs[self.parity], self.dp_size,
            opt._s1.data_ptr(), None if opt._s2 is None else opt._s2.data_ptr(), out.data_ptr(), self.numel, coef,
            opt._bad.data_ptr(), self.flags.data_ptr(), self.epoch_ctr.data_ptr(), self.timeout_ms,
            self.status.data_ptr(), stream,
        )
        _lib.check(rc, "po_step_predict_dp_dc")
        opt.step_count += 1
        self.parity ^= 1

    def check(self) -> None:
        """Raise if a fused update timed out waiting for a replica (syncs).
        The group is then poisoned: the kernel skipped that update (and would
        skip every later one), so further updates raise instead of silently
        advancing step counts over unchanged weights."""
        if self.poisoned or int(self.status.item()) != 0:
            self.poisoned = True
            raise RuntimeError("fused DP update timed out waiting for a replica's gradient signal")

    def close(self, dist=None, group=None) -> None:
        """Unmap the peers' buffers, free this replica's, release the NVLS
        object. Every replica must be done with the group: pass `dist` (and
        the group) to barrier first, or call it only after a barrier. The
        stage / optimizer must not use adopted buffers afterwards."""
        torch.cuda.synchronize(self.device)
        if dist is not None:
            dist.barrier(group=group)
        for pb in self._opened:
            pb.close()
        self._opened = []
        for b in self._ipc.values():
            b.free()
        self._ipc = {}
        if self._nvls is not None:
            _lib.check(self._lib.po_nvls_free(self._nvls), "po_nvls_free")
            self._nvls = None
        self.closed = True

    def _live(self) -> None:
        if self.closed:
            raise RuntimeError("fused DP group is closed")
        if self.poisoned:
            raise RuntimeError("fused DP group is poisoned: an earlier update timed out waiting for a replica")
