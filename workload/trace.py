"""Seeded request-arrival traces for the star workloads (BASELINE.json configs 4-5; SURVEY 8(d)
"Configs as concrete workloads").  Arrivals only -- no method arithmetic.

C5 bursty: per verifier, burst epochs form a Poisson process of rate `burst_rate_hz`; each burst
brings Geometric(mean `burst_mean`) requests at once; each request asks for Uniform{len_lo..len_hi}
emitted tokens.  C4 heterogeneous: fixed per-verifier cohorts (batch sizes and agreement knobs).
"""
from __future__ import annotations

import numpy as np

C4_BATCH = (32, 64, 128)          # per-verifier batch sizes of the heterogeneous 1 -> 3 star
C4_KAPPA = (3.0, 30.0, 300.0)     # per-verifier agreement (beta ~ 0.44 / 0.73 / 0.92)


def bursty_trace(n_verifiers: int, seconds: float, seed: int = 21622005,
                 burst_rate_hz: float = 20.0, burst_mean: float = 16.0, len_lo: int = 64,
                 len_hi: int = 512):
    """Compound-Poisson arrivals.  Returns, per verifier v = 1..n_verifiers, a list of
    (arrival_ms, length_tokens) sorted by time."""
    rng = np.random.default_rng(seed)
    out = {}
    for v in range(1, n_verifiers + 1):
        t, reqs = 0.0, []
        while True:
            t += rng.exponential(1000.0 / burst_rate_hz)
            if t >= seconds * 1000.0:
                break
            n = int(rng.geometric(1.0 / burst_mean))
            for _ in range(n):
                reqs.append((t, int(rng.integers(len_lo, len_hi + 1))))
        out[v] = reqs
    return out
