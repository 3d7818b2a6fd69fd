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
"""

from __future__ import annotations

import ctypes

import torch

from . import _lib


class FusedDPGroup:
    """Peer-mapped, double-buffered gradients of one stage's DP replicas."""

    def __init__(self, dist, group, dp_rank: int, dp_size: int, numel: int, device, timeout_ms: int = 60_000):
        from .ipc import IpcBuffer, open_peer

        if not 1 <= dp_size <= 8:
            raise ValueError(f"fused DP supports 1..8 replicas, got {dp_size}")
        self.dp_rank, self.dp_size, self.numel = dp_rank, dp_size, numel
        self.device = torch.device(device)
        self.timeout_ms = timeout_ms
        # node-shared (CUDA IPC) gradients and flags, mapped by each peer into
        # its own device (ipc.py)
        self._ipc = [IpcBuffer(numel, torch.float32, self.device) for _ in range(2)]
        self._ipc.append(IpcBuffer(dp_size, torch.int64, self.device))
        self.bufs = [self._ipc[0].tensor, self._ipc[1].tensor]
        self.flags = self._ipc[2].tensor
        self.status = torch.zeros(1, dtype=torch.int32, device=self.device)
        self.poisoned = False
        torch.cuda.synchronize(self.device)
        mine = [b.export() for b in self._ipc]
        handles = [None] * dp_size
        dist.all_gather_object(handles, mine, group=group)
        self.peers = []
        self._opened = []
        for r, h in enumerate(handles):
            if r == dp_rank:
                self.peers.append((self.bufs[0], self.bufs[1], self.flags))
            else:
                opened = [open_peer(x, self.device) for x in h]
                self._opened += opened
                self.peers.append(tuple(pb.tensor for pb in opened))
        # slot of THIS replica in every replica's flag array
        self.slots = torch.tensor([p[2].data_ptr() + 8 * dp_rank for p in self.peers], dtype=torch.int64,
                                  device=self.device)
        self.grad_ptrs = [(ctypes.c_void_p * dp_size)(*[self.peers[r][par].data_ptr() for r in range(dp_size)])
                          for par in (0, 1)]
        self.epoch = 0
        self.parity = 0
        self._lib = _lib.load()
        # CUDA-graph form (step_predict_dev): the epoch lives on the device
        self.epoch_ctr = torch.zeros(1, dtype=torch.int64, device=self.device)
        self._slot = None
        dist.barrier(group=group)

    @property
    def grad(self) -> torch.Tensor:
        """The buffer this replica's next backward must write into."""
        return self.bufs[self.parity]

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

    def _live(self) -> None:
        if self.poisoned:
            raise RuntimeError("fused DP group is poisoned: an earlier update timed out waiting for a replica")
