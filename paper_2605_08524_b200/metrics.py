"""Load-balance and utilisation figures (reference ``metrics.py:26-44``).

``attention_mfu`` keeps the reference's curve-normalised definition for the
analytic model; measured GPU runs report *raw* MFU against the measured B200
bf16 peak (``raw_mfu``), as BASELINE.md prescribes.
"""

from __future__ import annotations

from typing import Sequence

from .errors import ParameterError


def imbalance_ratio(loads: Sequence[float]) -> float:
    """(max - mean) / max; 0 for an all-zero load vector."""
    if len(loads) == 0:
        raise ParameterError("imbalance_ratio needs at least one worker")
    top = max(loads)
    if top <= 0:
        return 0.0
    return max(0.0, (top - sum(loads) / len(loads)) / top)


def attention_mfu(report, hw, n_workers: int, curve) -> float:
    if report.total_time <= 0:
        raise ParameterError("report has non-positive total_time")
    return report.total_flops / (n_workers * hw.peak_flops * report.total_time) / curve.saturation


def raw_mfu(total_flops: float, n_gpus: int, peak_flops: float, seconds: float) -> float:
    """FLOP_total / (N * peak * max-rank time) -- no curve normalisation."""
    if seconds <= 0:
        raise ParameterError("non-positive time")
    return total_flops / (n_gpus * peak_flops * seconds)
