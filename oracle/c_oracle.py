"""ctypes wrapper of oracle/c/optim_oracle.c — TEST/BASELINE INFRASTRUCTURE ONLY.

The C restatement is the multi-core CPU baseline bench.py times; it is pinned
to oracle/optim_ref.py (itself pinned to the reference) by tests/test_oracle.py.
"""

from __future__ import annotations

import ctypes
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "build" / "liboptim_oracle.so"
KIND = {"sgdm": 0, "adam": 1, "adamw": 2}


class OracleHP(ctypes.Structure):
    _fields_ = [
        ("kind", ctypes.c_int),
        ("momentum", ctypes.c_double),
        ("dampening", ctypes.c_double),
        ("weight_decay", ctypes.c_double),
        ("beta1", ctypes.c_double),
        ("beta2", ctypes.c_double),
        ("eps", ctypes.c_double),
        ("decoupled_decay", ctypes.c_double),
    ]


def build(force: bool = False) -> Path:
    src = HERE / "c" / "optim_oracle.c"
    if force or not LIB.exists() or LIB.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(HERE), "-B" if force else "all"], check=True)
    return LIB


_lib = None


def load() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not LIB.exists():
            build()
        lib = ctypes.CDLL(str(LIB))
        P = ctypes.c_void_p
        hp = ctypes.POINTER(OracleHP)
        lib.oracle_step.restype = ctypes.c_int64
        lib.oracle_step.argtypes = [hp, P, P, P, P, ctypes.c_int64, ctypes.c_double, ctypes.c_int64]
        lib.oracle_step_predict.restype = ctypes.c_int64
        lib.oracle_step_predict.argtypes = [
            hp, P, P, P, P, P, ctypes.c_int64, ctypes.c_double, ctypes.c_double, ctypes.c_int64
        ]
        lib.oracle_predict.restype = None
        lib.oracle_predict.argtypes = [hp, P, P, P, P, ctypes.c_int64, ctypes.c_double, ctypes.c_int64]
        lib.oracle_threads.restype = ctypes.c_int
        _lib = lib
    return _lib


def hp(kind: str, **kw) -> OracleHP:
    d = dict(momentum=0.9, dampening=0.0, weight_decay=5e-4, beta1=0.9, beta2=0.999, eps=1e-8,
             decoupled_decay=1e-2)
    d.update(kw)
    return OracleHP(KIND[kind], d["momentum"], d["dampening"], d["weight_decay"], d["beta1"],
                    d["beta2"], d["eps"], d["decoupled_decay"])


def _p(a):
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data


def step(h: OracleHP, w, g, s1, s2, lr, step_count) -> int:
    """In place on w/s1/s2 (float64); returns the non-finite count."""
    return load().oracle_step(ctypes.byref(h), _p(w), _p(g), _p(s1), _p(s2), w.size, lr, step_count)


def step_predict(h: OracleHP, w, g, s1, s2, w_hat, lr, lr_pred_times_s, step_count) -> int:
    return load().oracle_step_predict(ctypes.byref(h), _p(w), _p(g), _p(s1), _p(s2), _p(w_hat),
                                      w.size, lr, lr_pred_times_s, step_count)


def predict(h: OracleHP, w, s1, s2, w_hat, lr_times_s, step_count) -> None:
    load().oracle_predict(ctypes.byref(h), _p(w), _p(s1), _p(s2), _p(w_hat), w.size, lr_times_s,
                          step_count)


def threads() -> int:
    return int(load().oracle_threads())
