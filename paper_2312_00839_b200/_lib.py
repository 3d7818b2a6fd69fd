"""ctypes binding of the C-ABI in include/pipeoptim.h (libpipeoptim.so).

There is deliberately no CPU fallback: if the library is missing the product
path raises immediately (`LibraryMissing`), and every call checks the
returned status code.
"""

from __future__ import annotations

import contextlib
import ctypes
import threading
from pathlib import Path

from .build import LIB_PATH

PO_EINVAL = -22
PO_ENOSYS = -38
PO_SGDM, PO_ADAM, PO_ADAMW = 0, 1, 2
KIND_CODES = {"sgdm": PO_SGDM, "adam": PO_ADAM, "adamw": PO_ADAMW}

# Every symbol include/pipeoptim.h declares (tests check the .so exports them).
EXPORTS = (
    "po_abi_version",
    "po_strerror",
    "po_version_difference",
    "po_step",
    "po_predict",
    "po_step_predict",
    "po_direction",
    "po_axpy_predict",
    "po_coef_fill",
    "po_step_dc",
    "po_predict_dc",
    "po_step_predict_dc",
    "po_all_finite",
    "po_l2_discard",
    "po_loss_grad",
    "po_relu_bwd_bias",
    "po_splitk_bias_act",
    "po_act_bwd_bias",
    "po_dp_signal",
    "po_step_predict_dp",
    "po_dp_signal_dev",
    "po_step_predict_dp_dc",
    "po_dp_shard_range",
    "po_step_predict_dp_shard",
    "po_nvls_probe",
    "po_nvls_create",
    "po_nvls_open",
    "po_nvls_add_device",
    "po_nvls_bind",
    "po_nvls_size",
    "po_nvls_free",
    "po_head_supported",
    "po_head_fwd",
    "po_head_fwd_loss",
    "po_set_pdl",
    "po_set_gemm_tile",
    "po_get_gemm_tile",
    "po_get_pdl",
    "po_head_bwd",
    "po_wgrad_update_supported",
    "po_wgrad_update",
    "po_gemm_f32x3",
    "po_gemm_f32x3_available",
    "po_p2p_send",
    "po_p2p_recv",
    "po_ipc_alloc",
    "po_ipc_open",
    "po_ipc_close",
    "po_ipc_free",
    "po_lstm_cell_fwd",
    "po_lstm_cell_bwd",
    "po_lstm_cell_fwd_sk",
    "po_lstm_cell_bwd_sk",
)

PO_LOSS_MSE, PO_LOSS_SOFTMAX_XENT = 0, 1

PO_COEF_STEP, PO_COEF_PREDICT, PO_COEF_STEP_PREDICT = 0, 1, 2


class LibraryMissing(RuntimeError):
    """libpipeoptim.so is not built / not loadable: there is no fallback."""


class KernelError(RuntimeError):
    """A libpipeoptim call returned a non-zero status."""


class po_hparams(ctypes.Structure):
    _fields_ = [
        ("kind", ctypes.c_int32),
        ("_pad", ctypes.c_int32),
        ("momentum", ctypes.c_double),
        ("dampening", ctypes.c_double),
        ("weight_decay", ctypes.c_double),
        ("beta1", ctypes.c_double),
        ("beta2", ctypes.c_double),
        ("eps", ctypes.c_double),
        ("decoupled_decay", ctypes.c_double),
    ]


class po_launch(ctypes.Structure):
    _fields_ = [
        ("block", ctypes.c_int32),
        ("ctas_per_sm", ctypes.c_int32),
        ("vec", ctypes.c_int32),
        ("cache", ctypes.c_int32),
        ("unroll", ctypes.c_int32),
    ]


class po_coef(ctypes.Structure):
    _fields_ = [("lr", ctypes.c_float), ("c_pred", ctypes.c_float), ("inv_bc1", ctypes.c_float), ("inv_bc2", ctypes.c_float)]


class po_dp_multicast(ctypes.Structure):
    """Multicast (NVLS) addresses for po_step_predict_dp_shard (all NULL:
    peer loads / stores)."""

    _fields_ = [("grad", ctypes.c_void_p), ("w", ctypes.c_void_p), ("state1", ctypes.c_void_p),
                ("state2", ctypes.c_void_p), ("w_hat", ctypes.c_void_p)]


_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_D = ctypes.c_double
_HP = ctypes.POINTER(po_hparams)
_LA = ctypes.POINTER(po_launch)

_SIGNATURES = {
    "po_abi_version": (ctypes.c_int, []),
    "po_strerror": (ctypes.c_char_p, [ctypes.c_int]),
    "po_version_difference": (ctypes.c_int, [_I64, _I64, ctypes.POINTER(_I64)]),
    "po_step": (ctypes.c_int, [_HP, _P, _P, _P, _P, _P, _I64, _D, _I64, _P, _LA, _P]),
    "po_predict": (ctypes.c_int, [_HP, _P, _P, _P, _P, _I64, _D, _I64, _LA, _P]),
    "po_step_predict": (ctypes.c_int, [_HP, _P, _P, _P, _P, _P, _I64, _D, _D, _I64, _P, _LA, _P]),
    "po_direction": (ctypes.c_int, [_HP, _P, _P, _P, _I64, _I64, _LA, _P]),
    "po_axpy_predict": (ctypes.c_int, [_P, _P, _P, _I64, _D, _LA, _P]),
    "po_coef_fill": (ctypes.c_int, [_HP, ctypes.c_int32, _D, _D, _I64, _P]),
    "po_step_dc": (ctypes.c_int, [_HP, _P, _P, _P, _P, _I64, _P, _P, _LA, _P]),
    "po_predict_dc": (ctypes.c_int, [_HP, _P, _P, _P, _P, _I64, _P, _LA, _P]),
    "po_step_predict_dc": (ctypes.c_int, [_HP, _P, _P, _P, _P, _P, _I64, _P, _P, _LA, _P]),
    "po_l2_discard": (ctypes.c_int, [_P, _I64, _P]),
    "po_all_finite": (ctypes.c_int, [_P, _I64, _P, _I64, _P]),
    "po_loss_grad": (ctypes.c_int, [ctypes.c_int32, _P, _P, _I64, _I64, _P, _P, _P, _P]),
    "po_relu_bwd_bias": (ctypes.c_int, [_P, ctypes.c_int32, _P, _I64, _I64, _P, _P, ctypes.c_int32, _P]),
    "po_splitk_bias_act": (ctypes.c_int, [_P, ctypes.c_int32, _I64, _I64, _P, ctypes.c_int32, _P, _P, _P, _I64,
                                          _P]),
    "po_act_bwd_bias": (ctypes.c_int, [ctypes.c_int32, _P, ctypes.c_int32, _P, _I64, _I64, _P, _P, ctypes.c_int32,
                                       _P]),
    "po_dp_signal": (ctypes.c_int, [_P, ctypes.c_int32, _I64, _P]),
    "po_dp_signal_dev": (ctypes.c_int, [_P, ctypes.c_int32, _P, _P]),
    "po_step_predict_dp_dc": (ctypes.c_int, [_HP, _P, _P, ctypes.c_int32, _P, _P, _P, _I64, _P, _P, _P, _P, _I64,
                                             _P, _P]),
    "po_step_predict_dp": (ctypes.c_int, [_HP, _P, _P, ctypes.c_int32, _P, _P, _P, _I64, _D, _D, _I64, _P, _P, _I64,
                                          _I64, _P, _P]),
    "po_dp_shard_range": (ctypes.c_int, [_I64, ctypes.c_int32, ctypes.c_int32, ctypes.POINTER(_I64),
                                         ctypes.POINTER(_I64)]),
    "po_step_predict_dp_shard": (ctypes.c_int, [_HP, ctypes.c_int32, ctypes.c_int32, _P, _P, _P, _P, _P, _I64, _D, _D,
                                                _I64, _P, _P, _P, _P, _P, _I64, _P, _I64, _P, _P, _P]),
    "po_nvls_probe": (ctypes.c_int, [ctypes.c_int32, _I64, ctypes.POINTER(_I64)]),
    "po_nvls_create": (ctypes.c_int, [ctypes.c_int32, _I64, ctypes.POINTER(ctypes.c_int32),
                                      ctypes.POINTER(ctypes.c_void_p)]),
    "po_nvls_open": (ctypes.c_int, [ctypes.c_int32, ctypes.c_int32, _I64, ctypes.POINTER(ctypes.c_void_p)]),
    "po_nvls_add_device": (ctypes.c_int, [_P]),
    "po_nvls_bind": (ctypes.c_int, [_P, ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_void_p)]),
    "po_nvls_size": (_I64, [_P]),
    "po_nvls_free": (ctypes.c_int, [_P]),
    "po_head_supported": (ctypes.c_int, [_I64, _I64, _I64]),
    "po_head_fwd": (ctypes.c_int, [_P, _I64, _I64, _P, _P, ctypes.c_int32, _P, _P, _I64, _P]),
    "po_set_gemm_tile": (ctypes.c_int, [ctypes.c_int32]),
    "po_get_gemm_tile": (ctypes.c_int, []),
    "po_set_pdl": (ctypes.c_int, [ctypes.c_int32]),
    "po_get_pdl": (ctypes.c_int, []),
    "po_head_fwd_loss": (ctypes.c_int, [_P, _I64, _I64, _P, _P, ctypes.c_int32, _P, ctypes.c_int32, _P, _P, _P,
                                        _P, _P, _I64, _P]),
    "po_head_bwd": (ctypes.c_int, [_P, _I64, _I64, _P, ctypes.c_int32, _P, _P, _P, _P, ctypes.c_int32, _P]),
    "po_wgrad_update_supported": (ctypes.c_int, [_I64, _I64, _I64]),
    "po_wgrad_update": (ctypes.c_int, [_HP, _P, _I64, _P, _I64, _I64, _I64, _I64, _P, _P, _P, _P, _P, _D, _D, _I64,
                                       _P, _P, _I64, _P]),
    "po_gemm_f32x3": (ctypes.c_int, [ctypes.c_int32, ctypes.c_int32, _P, _I64, _I64, _P, _I64, _I64, _P, _I64, _I64,
                                     _I64, _I64, _P, _I64, _P]),
    "po_gemm_f32x3_available": (ctypes.c_int, []),
    "po_p2p_send": (ctypes.c_int, [_P, _I64, _P, _I64, ctypes.c_int32, _P, _P, _P, _I64, _P, _P]),
    "po_p2p_recv": (ctypes.c_int, [_P, _I64, ctypes.c_int32, _P, _I64, _P, _P, _P, _I64, _P, _P]),
    "po_ipc_alloc": (ctypes.c_int, [_I64, ctypes.POINTER(ctypes.c_void_p), ctypes.c_char_p]),
    "po_ipc_open": (ctypes.c_int, [ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p)]),
    "po_ipc_close": (ctypes.c_int, [_P]),
    "po_ipc_free": (ctypes.c_int, [_P]),
    "po_lstm_cell_fwd": (ctypes.c_int, [_P, _P, _P, _P, _P, _I64, _I64, _I64, _P]),
    "po_lstm_cell_bwd": (ctypes.c_int, [_P, _P, _P, _P, _I64, _P, _P, _P, _I64, _I64, _P]),
    "po_lstm_cell_fwd_sk": (ctypes.c_int, [_P, _P, ctypes.c_int32, _P, _P, _P, _P, _I64, _I64, _I64, _P]),
    "po_lstm_cell_bwd_sk": (ctypes.c_int, [_P, _P, _P, _P, _I64, _P, ctypes.c_int32, _P, _P, _I64, _I64, _P]),
}

_lock = threading.Lock()
_lib: ctypes.CDLL | None = None


def load(path: Path | str | None = None) -> ctypes.CDLL:
    """Load (once) and type the library; raises LibraryMissing if absent."""
    global _lib
    with _lock:
        if _lib is not None and path is None:
            return _lib
        p = Path(path) if path is not None else LIB_PATH
        if not p.exists():
            raise LibraryMissing(
                f"{p} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "(there is no CPU fallback for the PipeOptim kernels)"
            )
        try:
            lib = ctypes.CDLL(str(p))
        except OSError as exc:
            raise LibraryMissing(f"cannot load {p}: {exc}") from exc
        for name, (res, args) in _SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.po_abi_version() != 1:
            raise LibraryMissing(f"{p}: ABI version {lib.po_abi_version()} != 1")
        if path is None:
            _lib = lib
        return lib


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = load().po_strerror(rc).decode()
        if rc == PO_EINVAL:
            raise ValueError(f"{what}: {msg}")
        raise KernelError(f"{what}: {msg} (status {rc})")


def make_launch(block=0, ctas_per_sm=0, vec=0, cache=0, unroll=0):
    return po_launch(block, ctas_per_sm, vec, cache, unroll)


@contextlib.contextmanager
def pdl(on: bool):
    """Programmatic dependent launch of the short stream kernels on / off for
    the duration (po_set_pdl; process-wide, read when a kernel is launched or
    captured). Results are unchanged either way."""
    lib = load()
    old = lib.po_get_pdl()
    lib.po_set_pdl(1 if on else 0)
    try:
        yield
    finally:
        lib.po_set_pdl(old)
