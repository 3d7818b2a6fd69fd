"""Seeded datasets and the cycling batch stream — TEST ORACLE.

Restates pkg/src/pipesim/data.py (generators :66-115, the 80/20 interleave
split :49-57, BatchStream :118-148) so parity runs use the reference's exact
batches without importing it.
"""

from __future__ import annotations

import math

import numpy as np

from .rng_ref import Stream

TEACHER_HIDDEN = 8


def _split(x: np.ndarray, y: np.ndarray):
    """Every fifth sample (index % 5 == 4) is held out (data.py:49-57)."""
    held = (np.arange(x.shape[0]) % 5) == 4
    return x[~held], y[~held], x[held], y[held]


def _one_hot(labels: np.ndarray, classes: int) -> np.ndarray:
    out = np.zeros((labels.shape[0], classes))
    out[np.arange(labels.shape[0]), labels] = 1.0
    return out


def make_dataset(kind, n_samples, seed, input_dim=4, target_dim=1, n_classes=2, noise=0.0):
    """Returns (x_train, y_train, x_eval, y_eval, loss_kind) as float64 arrays."""
    if n_samples < 10:
        raise ValueError("n_samples must be >= 10")
    if kind == "synthetic-regression":
        x = Stream(seed, "dataset/x").normal(n_samples, input_dim)
        teacher = Stream(seed, "dataset/teacher")
        w1 = teacher.normal(input_dim, TEACHER_HIDDEN, scale=input_dim ** -0.5)
        w2 = teacher.normal(TEACHER_HIDDEN, target_dim, scale=TEACHER_HIDDEN ** -0.5)
        y = np.tanh(x @ w1) @ w2
        if noise > 0.0:
            y = y + noise * Stream(seed, "dataset/noise").normal(n_samples, target_dim)
        return (*_split(x, y), "mse")
    if kind == "two-spirals":
        if n_classes != 2:
            raise ValueError("two-spirals is a 2-class task")
        labels = np.arange(n_samples) % 2
        pos = np.arange(n_samples) // 2
        arm = max(1, (n_samples + 1) // 2 - 1)
        phi = 3.0 * math.pi * pos / arm
        r = 0.2 + 0.8 * phi / (3.0 * math.pi)
        ang = phi + labels * math.pi
        x = np.stack([r * np.cos(ang), r * np.sin(ang)], axis=1)
        if noise > 0.0:
            x = x + noise * Stream(seed, "dataset/noise").normal(n_samples, 2)
        return (*_split(x, _one_hot(labels, 2)), "softmax_xent")
    if kind == "tiny-classification":
        labels = np.arange(n_samples) % n_classes
        centers = Stream(seed, "dataset/centers").normal(n_classes, input_dim, scale=3.0)
        x = centers[labels] + Stream(seed, "dataset/points").normal(n_samples, input_dim, scale=0.5)
        if noise > 0.0:
            x = x + noise * Stream(seed, "dataset/noise").normal(n_samples, input_dim)
        return (*_split(x, _one_hot(labels, n_classes)), "softmax_xent")
    raise ValueError(f"unknown dataset kind: {kind!r}")


class Batches:
    """Cycles the training split in order, dropping the remainder (data.py:118-148).
    `batch(mb)` is 1-indexed."""

    def __init__(self, x_train: np.ndarray, y_train: np.ndarray, batch_size: int):
        if not 1 <= batch_size <= x_train.shape[0]:
            raise ValueError("bad batch_size")
        self.x, self.y, self.bs = x_train, y_train, batch_size
        self.steps_per_epoch = x_train.shape[0] // batch_size

    def batch(self, mb: int):
        if mb < 1:
            raise ValueError("mb is 1-indexed")
        lo = ((mb - 1) % self.steps_per_epoch) * self.bs
        return self.x[lo : lo + self.bs], self.y[lo : lo + self.bs]


def config1(seed: int = 0, n_samples: int = 3200, batch_size: int = 128):
    """SURVEY.md config 1 data: tiny-classification, 3072 inputs (CIFAR-10
    shaped), 10 classes, noise 32; returns (Batches, loss_kind)."""
    xt, yt, _, _, loss = make_dataset("tiny-classification", n_samples, seed, input_dim=3072,
                                      n_classes=10, noise=32.0)
    return Batches(xt, yt, batch_size), loss
