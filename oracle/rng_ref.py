"""Counter-based Philox streams keyed by SHA-256 of (seed, label) — TEST ORACLE.

Restates pkg/src/pipesim/linalg.py:141-167 so parity runs can rebuild the
reference's exact parameter init (stages.py:83-91) and datasets (data.py)
on the GPU box, where the reference is not installed. Pinned by
tests/test_oracle.py against the reference's golden RNG values
(pkg/tests/test_linalg.py:179-211) and against fixtures made by the reference.
"""

from __future__ import annotations

import hashlib

import numpy as np


def philox_key(seed: int, label: str) -> int:
    """128-bit little-endian key from sha256('pipesim:{seed}:{label}') (linalg.py:141-144)."""
    return int.from_bytes(hashlib.sha256(f"pipesim:{int(seed)}:{label}".encode()).digest()[:16], "little")


class Stream:
    """A labelled Philox stream; substreams extend the label with '/name'."""

    def __init__(self, seed: int, label: str = "root"):
        self.seed = int(seed)
        self.label = label
        self.gen = np.random.Generator(np.random.Philox(key=philox_key(self.seed, label)))

    def sub(self, name: str) -> "Stream":
        return Stream(self.seed, f"{self.label}/{name}")

    def normal(self, rows: int, cols: int, scale: float = 1.0) -> np.ndarray:
        return self.gen.standard_normal((rows, cols)) * float(scale)

    def uniform(self, rows: int, cols: int, low: float = 0.0, high: float = 1.0) -> np.ndarray:
        return self.gen.uniform(low, high, size=(rows, cols))


def layer_init(seed: int, index: int, in_dim: int, out_dim: int, root_label: str = "root/params"):
    """Reference init for global layer `index`: W ~ N(0,1)*in^-1/2 from the
    substream '<root>/params/layer-<index>', zero bias (stages.py:83-91 with the
    RngStream(seed).substream('params') root used by run_experiment)."""
    s = Stream(seed, f"{root_label}/layer-{index}")
    w = s.normal(in_dim, out_dim, scale=in_dim ** -0.5)
    return w, np.zeros((1, out_dim))
