"""Trace-driven star workloads (BASELINE.json configs 4-5): the seeded compound-Poisson bursty
trace (workload/trace.py) drives the star's FIFO scheduler (star.simulate_trace, host only).
Pinned to the Sec. 4.1 closed forms where the trace keeps every cohort busy, and to token
conservation; the C5 run reports busy fraction over time and per-verifier tokens/s."""
import math

import numpy as np
import pytest

from paper_2601_21622_b200 import star
from workload import C4_BATCH, bursty_trace


@pytest.mark.parametrize("N,S,Z", [(1, 1.0, 3.0), (2, 1.0, 3.0), (4, 1.0, 3.0), (3, 2.0, 1.0)])
def test_saturated_trace_follows_the_closed_form(N, S, Z):
    """Every verifier receives 128 requests that never finish at t = 0: each (single-slot) cohort
    is always active, so the trace-driven busy fraction is N S / (N S + T_idle), Eqs. 8-10."""
    tr = {v: [(0.0, 10**9)] * 128 for v in range(1, N + 1)}
    r = star.simulate_trace(tr, S, Z, 0.73, 5, n_slots=1, until_ms=4000.0)
    t_idle = max(0.0, Z - (N - 1) * S)
    assert r["busy_fraction"] == pytest.approx(N * S / (N * S + t_idle), abs=0.01)


def test_tokens_are_conserved_and_idle_verifiers_cost_nothing():
    """Run to completion: every request emits exactly its length.  A verifier with no arrivals
    issues no rounds (it never enters Q_in), so the star behaves as one with N - 1 verifiers."""
    tr = bursty_trace(3, 2.0, seed=11)
    r = star.simulate_trace(tr, 1.0, 3.0, [0.5, 0.8, 0.95], 7)
    total = sum(ln for v in tr for _, ln in tr[v])
    assert sum(r["tokens_per_s"]) * r["horizon_ms"] / 1000.0 == pytest.approx(total, rel=1e-9)
    assert r["completed_requests"] == sum(len(x) for x in tr.values())
    tr2 = {1: tr[1], 2: []}
    r2 = star.simulate_trace(tr2, 1.0, 3.0, 0.8, 7)
    r1 = star.simulate_trace({1: tr[1]}, 1.0, 3.0, 0.8, 7)
    assert r2["rounds"] == r1["rounds"] and r2["busy_fraction"] == pytest.approx(r1["busy_fraction"])


@pytest.mark.parametrize("N", [1, 3, 7])
def test_c5_bursty_trace_report(N):
    """C5: lambda_b = 20 bursts/s, Geometric(16) requests per burst, Uniform{64..512} tokens, 128
    active slots and two cohorts per verifier, beta = 0.73 (kappa = 30), k = 5.  With S = 1 ms and
    Z = 3 ms (Z/S = 3, the paper-calibrated ratio) the busy fraction grows with N
    toward the fully-loaded regime; every window's busy fraction is a fraction."""
    tr = bursty_trace(N, 3.0)
    r = star.simulate_trace(tr, 1.0, 3.0, 0.73, 5, n_slots=2)
    w = np.asarray(r["busy_per_window"])
    assert np.all((w >= 0) & (w <= 1 + 1e-9))
    assert len(r["tokens_per_s"]) == N and min(r["tokens_per_s"]) > 0
    if N == 7:
        assert r["busy_fraction"] > 0.9                     # 1 -> 7: the draft stays >= 90 % busy


def test_c4_heterogeneous_cohorts():
    """C4-style 1 -> 3 star with unequal batches (32/64/128 long requests) and betas
    (0.44 / 0.73 / 0.92): per-verifier token rates order with batch x (E[l] + 1), FIFO keeps the
    round counts equal (no verifier starves)."""
    tr = {v + 1: [(0.0, 10**9)] * C4_BATCH[v] for v in range(3)}
    r = star.simulate_trace(tr, 1.0, 3.0, [0.44, 0.73, 0.92], 7, n_slots=1, until_ms=3000.0)
    tps = r["tokens_per_s"]
    assert tps[0] < tps[1] < tps[2]
    el = [b * (1 - b ** 7) / (1 - b) for b in (0.44, 0.73, 0.92)]
    ratio = [t / (bs * (e + 1)) for t, bs, e in zip(tps, C4_BATCH, el)]
    assert max(ratio) / min(ratio) < 1.05                   # equal rounds per verifier
