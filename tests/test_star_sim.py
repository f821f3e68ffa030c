"""Round scheduler under the deterministic fake transport (sd_star_simulate),
pinned to the closed forms of PAPER.md Sec. 4.1:

  Eq. (Tidle)   T_idle   = max(0, Z - (N-1) S)             idle gap per iteration
  Eq. (Tgamma)  T_gamma  = N S + T_idle                      one iteration
  Eq. (busy)    Z <= (N-1) S  <=>  no idle gap (work-conserving M_q)
  P:336-340            N_full   = ceil(Z / S) + 1
  M_q load     busy     = N S / T_gamma
and T_wait = max(0, (N-1) S - Z): in the fully-loaded case every stream's cycle is
T_gamma_full = N S (Eq. P:224) = Z + T_wait + S.  Host only, no GPU.
"""
import math

import pytest

from paper_2601_21622_b200 import star
from paper_2601_21622_b200._lib import StarsdError

CASES = [(10.0, 30.0), (1.36, 30.6), (2.0, 0.0), (5.0, 12.5), (3.0, 9.0), (7.0, 1.0)]


@pytest.mark.parametrize("S,Z", CASES)
@pytest.mark.parametrize("N", [1, 2, 3, 4, 5, 8])
def test_busy_idle_wait_closed_forms(N, S, Z):
    sim = star.simulate(N, 1, S, Z, 4000)
    t_idle = max(0.0, Z - (N - 1) * S)
    t_gamma = N * S + t_idle
    assert sim["busy_fraction"] == pytest.approx(N * S / t_gamma, rel=1e-9, abs=1e-3)
    # mean gap between consecutive services; one iteration = N services -> T_idle = N * gap
    assert N * sim["mean_idle_ms"] == pytest.approx(t_idle, rel=2e-3, abs=1e-6)
    assert sim["mean_wait_ms"] == pytest.approx(max(0.0, (N - 1) * S - Z), rel=1e-6, abs=1e-6)
    # window: 4000 services, each S, plus one idle gap per N services
    assert sim["window_ms"] == pytest.approx(4000 * S + (4000 / N - 1) * t_idle, rel=2e-3)
    assert sim["rounds"] == 4000


@pytest.mark.parametrize("S,Z", CASES)
def test_n_full_is_the_first_zero_idle_N(S, Z):
    n_full = star.predicted(1, S, Z)["n_full"]
    assert n_full == math.ceil(Z / S) + 1
    assert star.simulate(n_full, 1, S, Z, 2000)["mean_idle_ms"] == 0.0
    if Z > 0 and n_full >= 2 and Z > (n_full - 2) * S:
        assert star.simulate(n_full - 1, 1, S, Z, 2000)["mean_idle_ms"] > 0.0


def test_paper_regime_Z30_S10():
    # Z = 30, S = 10: T_idle = 30, 20, 10, 0 for N = 1..4 and N_full = 4
    got = [n * star.simulate(n, 1, 10.0, 30.0, 3000)["mean_idle_ms"] for n in (1, 2, 3, 4)]
    assert got == pytest.approx([30.0, 20.0, 10.0, 0.0], rel=2e-3)
    assert star.predicted(4, 10.0, 30.0)["n_full"] == 4
    # busy grows by S/(S+Z) per added verifier until saturation (under-loaded regime)
    busy = [star.simulate(n, 1, 10.0, 30.0, 3000)["busy_fraction"] for n in range(1, 7)]
    assert busy == pytest.approx([0.25, 0.5, 0.75, 1.0, 1.0, 1.0], abs=1e-3)


@pytest.mark.parametrize("N,m", [(1, 2), (2, 2), (3, 3), (2, 4)])
def test_slots_act_as_independent_streams(N, m):
    # n_slots outstanding rounds per verifier = N*m closed-loop streams
    a = star.simulate(N, m, 4.0, 20.0, 3000)
    b = star.simulate(N * m, 1, 4.0, 20.0, 3000)
    for key in ("busy_fraction", "mean_idle_ms", "mean_wait_ms"):
        assert a[key] == pytest.approx(b[key], rel=1e-9, abs=1e-9)


def test_fifo_is_work_conserving():
    # with returns always pending (Z = 0) the draft never idles and nothing waits longer than
    # (N-1) S -- FIFO service order, no starvation of any verifier
    for n in (1, 2, 7):
        sim = star.simulate(n, 1, 3.0, 0.0, 1000)
        assert sim["busy_fraction"] == pytest.approx(1.0)
        assert sim["mean_wait_ms"] == pytest.approx((n - 1) * 3.0)


@pytest.mark.parametrize("args", [(0, 1, 1.0, 1.0, 10), (1, 0, 1.0, 1.0, 10),
                                  (1, 1, 0.0, 1.0, 10), (1, 1, 1.0, -1.0, 10),
                                  (1, 1, 1.0, 1.0, 0)])
def test_simulate_rejects_bad_arguments(args):
    with pytest.raises(StarsdError, match="INVALID_ARGUMENT"):
        star.simulate(*args)
