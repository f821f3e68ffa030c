"""Star analytics and admission (Sec. 4, Eqs. 3-11, P:153-248;
N_full / N_max), pinned to hand-derived values and validated by the fake-transport
discrete-event simulation (sd_star_simulate_ex) -- host only, no GPU.

  E[l_i]   = beta_i (1 - beta_i^d) / (1 - beta_i)      Eq. (3)
  T_idle   = max(0, Z - (N-1) S),  T_gamma = N S + T_idle          Eqs. (9)-(10)
  O_gamma  = E[l]_gamma / T_gamma,  O^(i) = E[l_i] / T_gamma        Eq. (11)
  N_full   = ceil(Z / S) + 1;  N_max = the largest N with O^(i) >= o_alone
"""
import numpy as np
import pytest

from paper_2601_21622_b200 import star
from paper_2601_21622_b200._lib import StarsdError


def test_closed_forms_on_a_hand_example():
    """beta = 0.8, d = 5: E[l] = 2.68928 (Eq. 3); S = 10 ms, Z = 30 ms (SPEC S:239-241
    regime): T_idle = 30/20/10/0 ms and T_gamma = 40/40/40/40 ms for N = 1..4, N_full = 4."""
    for N, t_idle in zip(range(1, 5), (30.0, 20.0, 10.0, 0.0)):
        p = star.analytics([0.8] * N, 5, 10.0, 30.0, 0.05)
        assert p["expected_accepted"] == pytest.approx(2.68928 * N, rel=1e-12)
        assert p["t_idle_ms"] == pytest.approx(t_idle)
        assert p["t_gamma_ms"] == pytest.approx(40.0)
        assert p["busy_fraction"] == pytest.approx(N * 10.0 / 40.0)
        assert p["throughput_per_ms"] == pytest.approx(2.68928 * N / 40.0)
        assert p["n_full"] == 4
    # beta = 1: every test accepted, E[l] = d (Eq. 3 limit); beta = 0: nothing accepted
    assert star.analytics([1.0], 5, 1.0, 1.0, 0.0)["expected_accepted"] == 5.0
    assert star.analytics([0.0], 5, 1.0, 1.0, 0.0)["expected_accepted"] == 0.0


def test_admission_bound_hand_example():
    """Same regime, o_alone = 0.05 tokens/ms: per-target O(N) = 2.68928 / T_gamma(N) is
    0.0672 for N <= 4 (T_gamma = 40), 0.0538 at N = 5 (50 ms), 0.0448 at N = 6 (60 ms) < 0.05,
    so N_max = 5 (by hand).  With o_alone above 2.68928 / 40, no N qualifies: N_max = 0."""
    assert star.analytics([0.8], 5, 10.0, 30.0, 0.05)["n_max"] == 5
    assert star.analytics([0.8], 5, 10.0, 30.0, 0.0672)["n_max"] == 4
    assert star.analytics([0.8], 5, 10.0, 30.0, 0.07)["n_max"] == 0


@pytest.mark.parametrize("beta,d,S,Z,o", [(0.8, 5, 10.0, 30.0, 0.05), (0.73, 7, 1.4, 4.0, 0.35),
                                          (0.9, 4, 2.0, 9.0, 0.12)])
def test_admission_bound_against_the_simulation(beta, d, S, Z, o):
    """The discrete-event simulation of the work-conserving FIFO star (one slot per target):
    every target's measured rounds x E[l] / window stays >= o_alone at N_max and falls below it
    at N_max + 1 -- the admission rule of P:343-345 holds on the simulated pipeline."""
    pred = star.analytics([beta], d, S, Z, o)
    el = pred["expected_accepted"]
    nmax = pred["n_max"]
    assert nmax >= 1
    for N, ok in ((nmax, True), (nmax + 1, False)):
        sim = star.simulate_ex([S] * N, [Z] * N, 1, 400 * N)
        per = np.array(sim["rounds_per_verifier"], float) * el / sim["window_ms"]
        assert (per.min() >= o * (1 - 1e-3)) == ok, (N, per, o)


def test_heterogeneous_star_under_and_fully_loaded():
    """C4-style heterogeneous star (per-verifier return times): under-loaded, each target cycles
    every S + Z_v, so its share of services is ~ 1/(S + Z_v); fully loaded, FIFO serves every
    target once per iteration (equal shares, no head-of-line blocking by the slow target)."""
    sim = star.simulate_ex([1.0, 1.0], [10.0, 30.0], 1, 4000)
    r = np.array(sim["rounds_per_verifier"], float)
    assert r[0] / r[1] == pytest.approx(31.0 / 11.0, rel=0.02)
    sim = star.simulate_ex([2.0, 2.0, 2.0], [1.0, 2.0, 3.0], 1, 3000)
    r = np.array(sim["rounds_per_verifier"], float)
    assert r.max() - r.min() <= 1 and sim["busy_fraction"] == pytest.approx(1.0)


def test_online_estimates_recover_S_Z_beta():
    """sd_sched_*: services of S = 2 ms, returns of Z = 6 ms and accept lengths drawn with a known
    per-position acceptance beta = 0.7 (k = 5, truncated geometric) -> the online estimates and
    the predicted N_full = ceil(6/2) + 1 = 4."""
    rng = np.random.default_rng(3)
    k, beta = 5, 0.7
    sc = star.Scheduler(2, k)
    t = 0.0
    for i in range(400):
        v = 1 + i % 2
        sc.service(v, t, t + 2.0)
        t += 2.0
        L = np.minimum(rng.geometric(1 - beta, 64) - 1, k)     # accepts before the first reject
        sc.observe(v, 6.0, L)
    p = sc.predict(0.0)
    assert p["service_ms"] == pytest.approx(2.0) and p["return_ms"] == pytest.approx(6.0)
    assert p["n_full"] == 4
    el = 2 * beta * (1 - beta ** k) / (1 - beta)
    assert p["expected_accepted"] == pytest.approx(el, rel=0.03)


def test_scheduler_fifo_and_misuse():
    sc = star.Scheduler(3, 4)
    for i, v in enumerate((2, 1, 3)):
        sc.push(v, 0, 7, float(i))
    assert [sc.pop(10.0)[0] for _ in range(3)] == [2, 1, 3]     # FIFO over Q_in
    assert sc.pop(10.0) is None
    with pytest.raises(StarsdError):
        sc.push(4, 0, 0, 0.0)                                   # no verifier 4
    with pytest.raises(StarsdError):
        star.Scheduler(2, 4).predict(0.1)                       # nothing observed yet
    with pytest.raises(StarsdError):
        star.analytics([0.5], 0, 1.0, 1.0, 0.1)                 # d >= 1
