"""Node-shared device buffers over CUDA IPC (NVLink / NVSwitch peer memory).

A buffer is a plain cudaMalloc allocation owned by one rank
(`IpcBuffer`), exported as a 64-byte handle; a neighbour maps it with
`open_peer` while ITS OWN device is current, so the mapping lives in the
device that dereferences it and peer access is enabled as needed (torch's
tensor-sharing path maps a handle into the OWNER's device context instead,
which is only correct when both processes share one GPU). Both sides see the
memory as a torch tensor (zero-copy, via __cuda_array_interface__) and as a
raw pointer for the kernels.
"""

from __future__ import annotations

import ctypes

import torch

from . import _lib

_TYPESTR = {torch.float32: "<f4", torch.int64: "<i8", torch.int32: "<i4"}


class _Cai:
    def __init__(self, ptr: int, numel: int, dtype: torch.dtype):
        self.__cuda_array_interface__ = {"shape": (numel,), "typestr": _TYPESTR[dtype], "data": (ptr, False),
                                         "version": 3, "strides": None}


def _wrap(ptr: int, numel: int, dtype: torch.dtype, device) -> torch.Tensor:
    return torch.as_tensor(_Cai(ptr, numel, dtype), device=device)


class IpcBuffer:
    """A zero-filled device buffer of `numel` `dtype` elements exportable to
    the other processes of the node."""

    def __init__(self, numel: int, dtype: torch.dtype, device):
        self.device = torch.device(device)
        self.numel, self.dtype = int(numel), dtype
        nbytes = max(1, self.numel) * torch.empty((), dtype=dtype).element_size()
        ptr = ctypes.c_void_p()
        handle = ctypes.create_string_buffer(64)
        with torch.cuda.device(self.device):
            _lib.check(_lib.load().po_ipc_alloc(nbytes, ctypes.byref(ptr), handle), "po_ipc_alloc")
        self.ptr = ptr.value
        self.handle = handle.raw
        self.tensor = _wrap(self.ptr, self.numel, dtype, self.device)

    def export(self) -> tuple:
        """Picklable description for `open_peer` in another process."""
        return (self.handle, self.numel, str(self.dtype).removeprefix("torch."))

    def free(self) -> None:
        if self.ptr:
            _lib.check(_lib.load().po_ipc_free(self.ptr), "po_ipc_free")
            self.ptr = 0


class PeerBuffer:
    """A neighbour's IpcBuffer mapped into this process's device."""

    def __init__(self, exported: tuple, device):
        handle, numel, dtype_name = exported
        self.device = torch.device(device)
        ptr = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            _lib.check(_lib.load().po_ipc_open(handle, ctypes.byref(ptr)), "po_ipc_open")
        self.ptr = ptr.value
        self.tensor = _wrap(self.ptr, numel, getattr(torch, dtype_name), self.device)

    def close(self) -> None:
        if self.ptr:
            _lib.check(_lib.load().po_ipc_close(self.ptr), "po_ipc_close")
            self.ptr = 0


def open_peer(exported: tuple, device) -> PeerBuffer:
    return PeerBuffer(exported, device)
