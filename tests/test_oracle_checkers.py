"""Pins of the oracle's checker half: the per-request trace the C-13 parity rule
reads (log-normalisers, a_j, u_acc, R, theta, C(t-1), C(t), the margins mu_a and mu_s),
sd_ref_sample_check, sd_ref_accept_probs and the zero-residual branch (C-6) of the sampling
distribution -- each against hand-derived values in tests/golden/worked_examples.json or a library
routine, never against the oracle itself."""
import json
import os

import numpy as np
import pytest
from scipy import special

import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")
WORKED = json.load(open(os.path.join(GOLD, "worked_examples.json")))
TOL = 1e-6     # the hand values are decimals stored as fp32 logits: ~1e-7 relative


def logits(p):
    with np.errstate(divide="ignore"):
        return np.log(np.asarray(p, np.float64)).astype(np.float32)


def chain_batch(ex, B):
    p = np.broadcast_to(np.stack([logits(r) for r in ex["p"]]), (B, len(ex["p"]), 3)).copy()
    q = np.broadcast_to(np.stack([logits(r) for r in ex["q"]]), (B, len(ex["q"]), 3)).copy()
    ids = np.broadcast_to(np.asarray(ex["ids"], np.int32), (B, len(ex["ids"]))).copy()
    return p, q, ids


def cell(cum, t):
    """(C(t-1), C(t)) of a hand CDF."""
    return (cum[t - 1] if t > 0 else 0.0), cum[t]


# ---------------------------------------------------------------- trace fields -------------
def test_trace_fields_on_the_inverse_cdf_hand_example():
    """Every trace field of the V=4 hand example: lam = 0 (logits are log-probs),
    a_0 = 0.25, u_acc from Philox, and at a rejection R = 0.4, theta = 0.4 u_smp, the CDF cell of
    the token from the hand residual [0, 0, .1, .3]; at acceptance the bonus CDF of p_1; mu_a =
    |u - 0.25| and mu_s = min(theta - C(t-1), C(t) - theta) / R."""
    ex = WORKED["inverse_cdf_hand"]
    B = 2000
    p = np.broadcast_to(np.stack([logits(ex["p0"]), logits(ex["p1"])]), (B, 2, 4)).copy()
    q = np.broadcast_to(logits(ex["q0"])[None], (B, 1, 4)).copy()
    ids = np.zeros((B, 1), np.int32)
    L, tok, st, tr = oracle.verify(p, q, ids, 1.0, seed=42, round=5, rid_base=0, trace=True)
    res_cum = np.cumsum(ex["residual"])
    nL = [0, 0]
    for b in range(B):
        t = tr[b]
        ua, _ = oracle.uniforms(42, 0, 5, b)
        assert abs(t.lam_p[0]) < TOL and abs(t.lam_q[0]) < TOL
        assert abs(t.a[0] - ex["a0"]) < TOL and abs(t.ell[0] - np.log(ex["a0"])) < TOL
        assert t.u_acc[0] == ua
        assert abs(t.mu_a - abs(ua - ex["a0"])) < TOL
        Lb = int(L[b])
        _, us = oracle.uniforms(42, Lb, 5, b)
        assert t.u_smp == us
        if Lb == 0:
            R, cum = ex["R"], res_cum
        else:
            R, cum = 1.0, np.asarray(ex["bonus_cdf"])
            assert abs(t.lam_p[1]) < TOL
        assert abs(t.R - R) < TOL and abs(t.theta - us * R) < TOL
        cp, ct = cell(cum, int(tok[b, Lb]))
        assert abs(t.C_prev - cp) < TOL and abs(t.C_tok - ct) < TOL
        assert abs(t.mu_s - min(us * R - cp, ct - us * R) / R) < 1e-5
        nL[Lb] += 1
    assert nL[0] > 1300 and nL[1] > 400         # Pr(L=0) = 0.75


def test_trace_and_decisions_on_the_accept_chain_hand_example():
    """V=3, k=3 hand chain: a = (.6, 1, .75); position 1 is accepted without a uniform; a rejection
    at 0 emits token 0, at 2 token 1; full acceptance draws the bonus from p_3; mu_a is the
    smallest |u_j - a_j| over the tests decided with a uniform."""
    ex = WORKED["accept_chain_hand"]
    B = 3000
    p, q, ids = chain_batch(ex, B)
    L, tok, st, tr = oracle.verify(p, q, ids, 1.0, seed=9, round=2, rid_base=100, trace=True)
    a = ex["a"]
    counts = np.zeros(4, int)
    for b in range(B):
        u = [oracle.uniforms(9, j, 2, 100 + b)[0] for j in range(3)]
        want_L, mu = 3, 1.0
        for j in range(3):
            if a[j] < 1.0:
                mu = min(mu, abs(u[j] - a[j]))
                if u[j] >= a[j]:
                    want_L = j
                    break
        assert L[b] == want_L and st[b] == 0
        t = tr[b]
        assert abs(t.mu_a - mu) < TOL
        for j in range(min(want_L + 1, 3)):
            assert abs(t.a[j] - a[j]) < TOL and abs(t.ell[j] - ex["ell"][j]) < TOL
        _, us = oracle.uniforms(9, want_L, 2, 100 + b)
        if want_L == 3:
            cum, R = np.asarray(ex["bonus_cdf"]), 1.0
        else:
            cum, R = np.cumsum(ex["residual_at"][str(want_L)]), ex["R_at"][str(want_L)]
        assert abs(t.R - R) < TOL and abs(t.theta - us * R) < TOL
        tk = int(tok[b, want_L])
        if want_L == 0:
            assert tk == 0
        elif want_L == 2:
            assert tk == 1
        else:
            assert tk == int(np.argmax(cum > us))
        cp, ct = cell(cum, tk)
        assert abs(t.C_prev - cp) < TOL and abs(t.C_tok - ct) < TOL
        counts[want_L] += 1
    assert counts[1] == 0                       # a_1 = 1: never rejected
    frac = counts / B                           # Pr(L = 0, 2, 3) = .4, .6 x .25 = .15, .45
    assert abs(frac[0] - 0.4) < 0.05 and abs(frac[2] - 0.15) < 0.04 and abs(frac[3] - 0.45) < 0.05


# ---------------------------------------------------------------- sample_check -------------
@pytest.mark.parametrize("L", [0, 1, 2, 3])
def test_sample_check_cells_are_the_hand_cdf(L):
    """sd_ref_sample_check at a FORCED accept length: the hand residual (or bonus) CDF cell of
    every token, R and theta = u_smp(L) R."""
    ex = WORKED["accept_chain_hand"]
    p, q, ids = chain_batch(ex, 4)
    if L == 3:
        cum, R = np.asarray(ex["bonus_cdf"]), 1.0
    else:
        cum, R = np.cumsum(ex["residual_at"][str(L)]), ex["R_at"][str(L)]
    for b in range(4):
        _, us = oracle.uniforms(3, L, 8, 50 + b)
        for t in range(3):
            Cp, Ct, Rv, th = oracle.sample_check(p, q, ids, b, L, t, 1.0, seed=3, round=8,
                                                 rid_base=50)
            cp, ct = cell(cum, t)
            assert abs(Cp - cp) < TOL and abs(Ct - ct) < TOL
            assert abs(Rv - R) < TOL and abs(th - us * R) < TOL


def test_sample_check_zero_residual_falls_back_to_p():
    """C-6: identical rows at the forced position have no residual mass; the cells are those of
    p itself (hand CDF .5, .8, 1) and R = sum p = 1."""
    ex = WORKED["accept_chain_hand"]
    z = logits(ex["identical_rows"])
    p = np.stack([z, z])[None].copy()           # k = 1: p_0, p_1
    q = z[None, None].copy()
    ids = np.zeros((1, 1), np.int32)
    cum = ex["identical_rows_cdf"]
    for t in range(3):
        Cp, Ct, R, th = oracle.sample_check(p, q, ids, 0, 0, t, 1.0, seed=1, round=0, rid_base=0)
        cp, ct = cell(cum, t)
        assert abs(Cp - cp) < TOL and abs(Ct - ct) < TOL and abs(R - 1.0) < TOL


# ---------------------------------------------------------------- accept_probs -------------
def test_accept_probs_are_the_hand_ratios_and_w0_uniforms():
    """sd_ref_accept_probs: a_j = min(1, p_j(x_j)/q_j(x_j)) at EVERY position (no early stop):
    (.6, 1, .75) by hand; u_j = u24(w0) of Philox counter (j, round, rid) (C-8)."""
    ex = WORKED["accept_chain_hand"]
    p, q, ids = chain_batch(ex, 3)
    for b in range(3):
        a, u = oracle.accept_probs(p, q, ids, b, 1.0, seed=77, round=4, rid_base=9)
        np.testing.assert_allclose(a, ex["a"], atol=TOL)
        for j in range(3):
            w = oracle.philox([j, 4, 9 + b, 0], [77, 0])
            assert u[j] == (int(w[0]) >> 8) / 2.0 ** 24


# ---------------------------------------------------------------- C-6 inside verify --------
def test_verify_zero_residual_samples_from_p():
    """A rejection whose fp64 residual vanishes: q equals p except at the draft token x, whose
    q logit is larger by 1 while p(x) ~ e^-60, so the log-normalisers agree to fp64 precision,
    every p(y) - q(y) with y != x is exactly 0 and a = p(x)/q(x) = e^-1.  At a rejection the step
    must flag SD_FAULT_ZERO_RESIDUAL and sample from p_0 itself: the token is the inverse CDF of the
    library softmax (scipy) at theta = u_smp(0) * sum p, R = sum p = 1."""
    V, B = 50, 600
    rng = np.random.default_rng(5)
    zp = rng.normal(0.0, 1.0, (B, 2, V)).astype(np.float32)
    x = rng.integers(0, V, B).astype(np.int32)
    zp[np.arange(B), 0, x] = -60.0
    zq = zp[:, :1].copy()
    zq[np.arange(B), 0, x] = -59.0
    ids = x[:, None].copy()
    L, tok, st, tr = oracle.verify(zp, zq, ids, 1.0, seed=13, round=1, rid_base=0, trace=True)
    rej = 0
    for b in range(B):
        ua, us = oracle.uniforms(13, 0, 1, b)
        assert abs(tr[b].a[0] - np.exp(-1.0)) < 1e-12
        if ua >= np.exp(-1.0):
            assert L[b] == 0 and st[b] & oracle.FAULT_ZERO_RESIDUAL
            pr = special.softmax(zp[b, 0].astype(np.float64))
            C = np.cumsum(pr)
            th = us * pr.sum()
            if np.min(np.abs(C - th)) < 1e-12:
                continue
            assert tok[b, 0] == int(np.searchsorted(C, th, side="right"))
            assert abs(tr[b].R - 1.0) < 1e-12
            rej += 1
        else:
            assert L[b] == 1 and not st[b] & oracle.FAULT_ZERO_RESIDUAL
    assert rej > 300


# ---------------------------------------------------------------- draft sampler (NEXT-2) ---
def test_draft_sampler_hand_cdf_and_counter_domain():
    """sd_ref_draft_sample on the hand row q = [.1,.2,.3,.4]: x = the first y whose hand CDF
    (.1,.3,.6,1) exceeds u = u24(w1) of the Philox counter (0, round, 2^63 + (rid_base + b) k + j)
    (reading D-1), and log q(x) = log of the hand probability; k = 3 positions share the
    row but use their own counters."""
    ex = WORKED["inverse_cdf_hand"]
    B, k = 300, 3
    q = np.broadcast_to(logits(ex["p0"]), (B, k, 4)).copy()
    ids, logq, mu, st = oracle.draft_sample(q, 1.0, seed=21, round=6, rid_base=40)
    cdf = np.asarray(ex["bonus_cdf"])
    for b in range(B):
        for j in range(k):
            _, u = oracle.uniforms(21, 0, 6, (1 << 63) + (40 + b) * k + j)
            if np.min(np.abs(cdf - u)) < 1e-6:
                continue
            x = int(np.argmax(cdf > u))
            assert ids[b, j] == x and abs(logq[b, j] - np.log(ex["p0"][x])) < TOL
    assert np.all(st == 0)


def test_draft_sampler_follows_the_library_softmax():
    """20000 draws from one V = 50 row at T = 0.7: the histogram matches scipy's softmax(z/T)
    (G-test), greedy (T = 0) is numpy's argmax with the lowest index on ties, faulty rows give -1."""
    from scipy import stats
    rng = np.random.default_rng(8)
    z = rng.normal(0, 1.5, 50).astype(np.float32)
    q = np.broadcast_to(z, (20000, 1, 50)).copy()
    ids, logq, mu, st = oracle.draft_sample(q, 0.7, seed=3, round=1)
    pr = special.softmax(z.astype(np.float64) / 0.7)
    obs = np.bincount(ids[:, 0], minlength=50)
    keep = pr * 20000 > 5
    g = 2 * np.sum(obs[keep] * np.log(np.maximum(obs[keep], 1) / (20000 * pr[keep])))
    assert stats.chi2.sf(g, keep.sum() - 1) > 1e-4
    np.testing.assert_allclose(logq[:, 0], np.log(pr[ids[:, 0]]), atol=1e-9)
    zt = z.copy()
    zt[[7, 30]] = zt.max() + 1.0                      # a tie for the maximum: lowest index wins
    g0 = oracle.draft_sample(zt[None, None].copy(), 0.0)[0]
    assert g0[0, 0] == int(np.argmax(zt)) == 7
    bad = np.stack([z, z]).copy()[None]
    bad[0, 0, 3] = np.nan
    bad[0, 1, :] = -np.inf
    ids, _, _, st = oracle.draft_sample(bad, 1.0)
    assert list(ids[0]) == [-1, -1] and list(st[0]) == [oracle.FAULT_NONFINITE, oracle.FAULT_EMPTY_ROW]
