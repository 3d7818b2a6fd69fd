"""Exception types mirroring the reference (pkg/src/pipesim/linalg.py:15-20,
stages.py:27-28, schedule.py:31-32)."""


class NumericError(RuntimeError):
    """Non-finite value produced where a finite one is required (linalg.py:19-20)."""


class DimensionError(ValueError):
    """Shape mismatch; the message names both shapes (linalg.py:15-16)."""


class StashError(RuntimeError):
    """Activation stash misuse: duplicate store or missing entry (stages.py:27-28)."""


class TimelineError(ValueError):
    """A timeline violates the schedule invariants (schedule.py:31-32)."""
