"""PipeOptim (arXiv 2312.00839) hot path, B200-native.

Optimizer-dependent weight prediction + optimizer step kernels (sm_100a, C-ABI
in include/pipeoptim.h), per-stage version bookkeeping and the 1F1B stage
runner, behind the reference simulator's Python API (pkg/src/pipesim).
"""

from .errors import DimensionError, NumericError, StashError, TimelineError
from .optim import (
    OPTIMIZER_KINDS,
    FlatLayout,
    FlatParams,
    OptimizerConfig,
    OptimizerState,
    predict_weights,
    version_difference,
)

__all__ = [
    "DimensionError",
    "NumericError",
    "StashError",
    "TimelineError",
    "OPTIMIZER_KINDS",
    "FlatLayout",
    "FlatParams",
    "OptimizerConfig",
    "OptimizerState",
    "predict_weights",
    "version_difference",
]
