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


def latency_stats(values) -> dict:
    """count, mean and the nearest-rank p50/p90/p95/p99 of a list (MetricsCollector's
    latency_stats, metrics.cpp:159-190), in the values' unit."""
    n = len(values)
    return {"count": n, "mean": float(sum(values) / n) if n else 0.0,
            **{f"p{int(q * 100)}": float(percentile(values, q)) for q in (0.5, 0.9, 0.95, 0.99)}}


def poisson_arrivals(n: int, qps: float, seed: int = 1):
    """Arrival times (us) of n requests of a Poisson process at `qps` requests/s: exponential
    gaps from a seeded generator, the first request at t = 0."""
    import numpy as np
    rng = np.random.default_rng(seed)
    gaps = rng.exponential(1e6 / qps, size=n)
    gaps[0] = 0.0
    return np.round(np.cumsum(gaps)).astype(np.int64)


def load_arrivals(path: str):
    """The reference's arrivals file (save_arrivals / load_arrivals, workload.hpp:56-59):
    a header, then `t_us,app_id,prompt_tokens,output_tokens[,prefix_group,prefix_tokens]` rows.
    Returns a list of (t_us, app_id, prompt_tokens, output_tokens)."""
    rows = []
    with open(path) as f:
        next(f, None)
        for line in f:
            parts = line.strip().split(",")
            if len(parts) < 4:
                continue
            rows.append(tuple(int(p) for p in parts[:4]))
    return rows


def serving_report(arrival_us, first_us, done_us, generated) -> dict:
    """build_report's request section (metrics.cpp:159-190) from live time stamps: latency =
    completion - arrival, ttft = first token - arrival (ms here), throughput = generated tokens /
    drain (the last completion, on the same clock as the arrivals)."""
    lat = [(d - a) / 1e3 for a, d in zip(arrival_us, done_us) if d >= 0]
    ttft = [(f - a) / 1e3 for a, f in zip(arrival_us, first_us) if f >= 0]
    drain_s = float(max(done_us)) / 1e6 if len(done_us) else 0.0
    return {"requests": len(arrival_us), "completed": len(lat),
            "latency_ms": latency_stats(lat), "ttft_ms": latency_stats(ttft),
            "drain_s": drain_s,
            "throughput_tokens_per_s": float(tokens_per_s(int(generated), drain_s))}
