"""Serving metrics with the reference's definitions (proj/core/src/metrics.cpp)."""
from __future__ import annotations

import math


def percentile(values, q: float) -> float:
    """Nearest-rank percentile: the ceil(q*n)-th smallest value (metrics.cpp:30-38);
    0.0 for no values; q must lie in (0, 1]."""
    if len(values) == 0:
        return 0.0
    if not (0.0 < q <= 1.0):
        raise ValueError("percentile q out of (0, 1]")
    v = sorted(values)
    rank = math.ceil(q * len(v))
    rank = min(max(rank, 1), len(v))
    return v[rank - 1]


def tokens_per_s(generated_tokens: int, drain_s: float) -> float:
    """Throughput = generated tokens / drain time (metrics.cpp:186-188)."""
    return generated_tokens / drain_s if drain_s > 0 else 0.0
