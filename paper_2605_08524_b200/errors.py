"""Exception taxonomy of the FCP control plane and GPU data plane.

Mirrors the reference hierarchy (``pkg/src/blocksched/errors.py:4-31``) so that
callers catching ``SchedulerError`` / ``ParameterError`` / ``InfeasibleError``
keep working unchanged.  The data plane adds ``NativeError`` for a failing
C-ABI status (a CUDA / NCCL failure inside ``libfcpb.so``).
"""

from __future__ import annotations


class SchedulerError(Exception):
    """Root of every error this package raises on purpose."""


class ParameterError(SchedulerError, ValueError):
    """A caller-supplied value breaks a documented precondition."""


class TraceFormatError(SchedulerError, ValueError):
    """Malformed trace file; ``line`` holds the 1-based offending line."""

    def __init__(self, message: str, line: int | None = None):
        self.line = line
        super().__init__(message if line is None else f"line {line}: {message}")


class InfeasibleError(SchedulerError, RuntimeError):
    """The constraints admit no schedule (e.g. the per-worker token cap)."""


class ConsistencyError(SchedulerError, RuntimeError):
    """Two artefacts that must describe the same batch disagree."""


class InternalError(SchedulerError, RuntimeError):
    """A should-never-happen invariant broke."""


class NativeError(SchedulerError, RuntimeError):
    """The CUDA extension returned a non-zero status (see ``fcpb_last_error``)."""
