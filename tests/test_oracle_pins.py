"""Pins of the CPU oracle against what the paper and the mathematics fix (no GPU needed).

Every test compares the oracle with something that is NOT the oracle: printed values
(tests/golden/, cited), known-answer vectors, library routines (scipy softmax, torch.argmax),
exact enumeration against the target distribution (losslessness), closed forms (Eq. 1, Eq. 3,
Lemma 1) and brute force on tiny inputs.
"""
import itertools
import json
import os

import numpy as np
import pytest
from scipy import special, stats

import oracle
from workload import make_batch, make_tiny_tables, tiny_batch, bf16_bits

GOLD = os.path.join(os.path.dirname(__file__), "golden")
WORKED = json.load(open(os.path.join(GOLD, "worked_examples.json")))


def logits(p):
    with np.errstate(divide="ignore"):
        return np.log(np.asarray(p, np.float64)).astype(np.float32)


def sm(z, T=1.0):
    """library softmax (scipy) of fp32 logits in fp64 -- independent of the oracle"""
    return special.softmax(np.asarray(z, np.float64) / T, axis=-1)


# ---------------------------------------------------------------- Philox (C-8) -------------
def test_philox_known_answer_vectors():
    rows = [l.split() for l in open(os.path.join(GOLD, "philox4x32_10_kat.txt"))
            if l.strip() and not l.startswith("#")]
    assert len(rows) == 3
    for r in rows:
        v = [int(x, 16) for x in r]
        out = oracle.philox(v[0:4], v[4:6])
        assert list(out) == v[6:10]


def test_u24_grid_and_counter_layout():
    # u24(w) = (w >> 8) 2^-24: check by a direct Philox call with the documented counter layout
    seed, j, rnd, rid = 0x1234567890ABCDEF, 3, 0x1_0000_0007, 0xDEADBEEF_00000011
    w = oracle.philox([j, rnd & 0xFFFFFFFF, rid & 0xFFFFFFFF, rid >> 32],
                      [seed & 0xFFFFFFFF, seed >> 32])
    ua, us = oracle.uniforms(seed, j, rnd, rid)
    assert ua == (int(w[0]) >> 8) / 2**24 and us == (int(w[1]) >> 8) / 2**24
    assert 0.0 <= ua < 1.0 and 0.0 <= us < 1.0


def test_uniform_marginals_ks():
    """P11: u_acc and u_smp marginals are uniform; w0/w1 uncorrelated."""
    n = 20000
    ua = np.empty(n)
    us = np.empty(n)
    for i in range(n):
        ua[i], us[i] = oracle.uniforms(21622, i % 7, i // 7, 99)
    assert stats.kstest(ua, "uniform").pvalue > 1e-3
    assert stats.kstest(us, "uniform").pvalue > 1e-3
    assert abs(np.corrcoef(ua, us)[0, 1]) < 4.0 / np.sqrt(n)


# ---------------------------------------------------------------- Eq. (1) -------------------
@pytest.mark.parametrize("ex", WORKED["beta_eq1"])
def test_beta_worked_examples(ex):
    assert abs(oracle.beta(logits(ex["p"]), logits(ex["q"])) - ex["beta"]) < 1e-7


def test_beta_equals_one_minus_tv():
    """P2: sum_x min(p,q) = 1 - 1/2 sum |p - q|, with p, q from scipy softmax."""
    rng = np.random.default_rng(1)
    for _ in range(1000):
        V = int(rng.integers(2, 65))
        zp = rng.normal(0, 2, V).astype(np.float32)
        zq = rng.normal(0, 2, V).astype(np.float32)
        T = float(rng.choice([0.5, 1.0, 1.7]))
        tv = 0.5 * np.abs(sm(zp, T) - sm(zq, T)).sum()
        assert abs(oracle.beta(zp, zq, T) - (1.0 - tv)) < 1e-12


def test_softmax_matches_library():
    rng = np.random.default_rng(2)
    for T in (0.3, 1.0, 2.5):
        z = rng.normal(0, 3, 500).astype(np.float32)
        z[::17] = -np.inf
        np.testing.assert_allclose(oracle.softmax(z, T), sm(z, T), rtol=1e-13, atol=1e-300)


# ---------------------------------------------------------------- losslessness --------------
def test_lossless_v2_worked_example():
    """V=2, p=[.7,.3], q=[.4,.6], d=1 -> emitted distribution [.7,.3]."""
    ex = WORKED["lossless_v2"]
    zp, zq = logits(ex["p"]), logits(ex["q"])
    q = sm(zq)
    emitted = np.zeros(2)
    for x in (0, 1):
        p_rows = np.stack([zp, zp])[None]
        out = oracle.outcome_dist(p_rows, zq[None, None], np.array([[x]]), 1.0)[0]
        emitted += q[x] * out[0]            # rejected at 0: the correction is emitted first
        emitted[x] += q[x] * out[1].sum()   # accepted: x is emitted first
    np.testing.assert_allclose(emitted, sm(zp), atol=1e-15)
    np.testing.assert_allclose(emitted, ex["emitted"], atol=1e-7)


def _completed_joint(P, Q, V, k, T):
    """Exhaustive C1 check: distribution of the k+1 tokens obtained by one verify round
    (over all V^k draft paths, weighted by the draft's own probability) completed by target
    sampling, and the plain autoregressive target joint over k+1 tokens."""
    paths = np.array(list(itertools.product(range(V), repeat=k)), np.int32)
    p, q = tiny_batch(P, Q, paths)
    out = oracle.outcome_dist(p, q, paths, T)                    # [V^k, k+1, V]
    w = np.ones(len(paths))
    for j in range(k):
        w *= sm(q[np.arange(len(paths)), j], T)[np.arange(len(paths)), paths[:, j]]
    # mass[n] over emitted sequences of length n (index = base-V number)
    mass = [np.zeros(V ** n) for n in range(k + 2)]
    for L in range(k + 1):
        pre = np.zeros(len(paths), np.int64)
        for i in range(L):
            pre = pre * V + paths[:, i]
        idx = (pre[:, None] * V + np.arange(V)[None, :]).ravel()
        np.add.at(mass[L + 1], idx, (w[:, None] * out[:, L, :]).ravel())
    # complete every emitted prefix with target sampling (p conditioned on the prefix)
    for n in range(1, k + 1):
        pn = np.stack([sm(P[s], T) for s in itertools.product(range(V), repeat=n)])
        mass[n + 1] += (mass[n][:, None] * pn).ravel()
    target = np.ones(1)
    for n in range(k + 1):
        pn = np.stack([sm(P[s], T) for s in itertools.product(range(V), repeat=n)])
        target = (target[:, None] * pn).ravel()
    return mass[k + 1], target


@pytest.mark.parametrize("T", [1.0, 0.7])
def test_lossless_exhaustive_tiny(T):
    """P5 / SURVEY C1: V=8, k=4, prefix-conditioned tables, all 8^4 draft paths: the emitted
    tokens are distributed exactly as autoregressive sampling from p."""
    P, Q = make_tiny_tables(V=8, k=4, seed=21622001)
    spec, target = _completed_joint(P, Q, 8, 4, T)
    assert abs(spec.sum() - 1.0) < 1e-12
    assert 0.5 * np.abs(spec - target).sum() < 1e-12


def test_literal_alg2_rule_is_not_lossless():
    """Reading C-1: the literal test of P:731 (accept iff r <= p(x), no q) would emit
    [41/50, 9/50] on the S:108 example; the oracle emits [7/10, 3/10]."""
    p = np.array([0.7, 0.3]); q = np.array([0.4, 0.6])
    lit = np.zeros(2)
    for x in (0, 1):
        resid = np.maximum(p - q, 0); resid /= resid.sum()
        lit[x] += q[x] * p[x]
        lit += q[x] * (1 - p[x]) * resid
    assert np.allclose(lit, [41 / 50, 9 / 50])
    assert not np.allclose(lit, p, atol=1e-3)


@pytest.mark.parametrize("T", [1.0, 0.6])
def test_step_by_step_matches_exact_outcome_distribution(T):
    """The step-by-step verify (Philox uniforms) against the uniforms-integrated outcome
    distribution: chi-square over (L, token) for one fixed request replicated over rids."""
    rng = np.random.default_rng(5)
    V, k, B = 6, 3, 60000
    zp = rng.normal(0, 1.5, (1, k + 1, V)).astype(np.float32)
    zq = rng.normal(0, 1.5, (1, k, V)).astype(np.float32)
    ids = np.array([[1, 4, 2]], np.int32)
    exact = oracle.outcome_dist(zp, zq, ids, T)[0].ravel()
    L, tok, st = oracle.verify(np.repeat(zp, B, 0), np.repeat(zq, B, 0), np.repeat(ids, B, 0),
                               T, seed=777, round=3, rid_base=1000, n_threads=4)
    assert np.all(st == 0)
    cell = L * V + tok[np.arange(B), L]
    obs = np.bincount(cell, minlength=(k + 1) * V)
    keep = exact * B > 5
    chi2 = ((obs[keep] - B * exact[keep]) ** 2 / (B * exact[keep])).sum()
    assert obs[~keep].sum() <= max(10, 3 * B * exact[~keep].sum() + 10)
    assert stats.chi2.sf(chi2, keep.sum() - 1) > 1e-4


@pytest.mark.parametrize("T", [1.0, 0.6])
def test_first_token_monte_carlo_lossless(T):
    """Draft ids drawn from q (x ~ q): the first emitted token follows p_0 (chi-square)."""
    rng = np.random.default_rng(6)
    V, k, B = 5, 2, 80000
    zp = rng.normal(0, 1.0, (k + 1, V)).astype(np.float32)
    zq = rng.normal(0, 1.0, (k, V)).astype(np.float32)
    qs = sm(zq, T)
    ids = np.stack([rng.choice(V, B, p=qs[j]) for j in range(k)], 1).astype(np.int32)
    L, tok, _ = oracle.verify(np.broadcast_to(zp, (B, k + 1, V)).copy(),
                              np.broadcast_to(zq, (B, k, V)).copy(), ids, T, seed=9,
                              n_threads=4)
    first = tok[:, 0]
    obs = np.bincount(first, minlength=V)
    exp = B * sm(zp[0], T)
    chi2 = ((obs - exp) ** 2 / exp).sum()
    assert stats.chi2.sf(chi2, V - 1) > 1e-4


# ---------------------------------------------------------------- Eq. (3), Lemma 1 ----------
@pytest.mark.parametrize("ex", WORKED["expected_accept_length_eq3"])
def test_expected_accept_length_closed_form(ex):
    """Rows with acceptance exactly beta per position (p = [b, 1-b], q = [1, 0], x = 0):
    E[L] = sum_j Pr(L >= j) (Lemma 1) = beta(1-beta^d)/(1-beta) (Eq. 3)."""
    b, d = ex["beta"], ex["d"]
    zp = logits([b, 1 - b]) if 0 < b < 1 else (logits([1.0, 0.0]) if b == 1 else logits([0.0, 1.0]))
    zq = logits([1.0, 0.0])
    p = np.broadcast_to(zp, (1, d + 1, 2)).copy()
    q = np.broadcast_to(zq, (1, d, 2)).copy()
    out = oracle.outcome_dist(p, q, np.zeros((1, d), np.int32), 1.0)[0]
    pL = out.sum(-1)
    assert abs(pL.sum() - 1) < 1e-12
    EL = (np.arange(d + 1) * pL).sum()
    assert abs(EL - ex["E_l"]) < 1e-6
    tail = [pL[j:].sum() for j in range(1, d + 1)]
    assert abs(sum(tail) - EL) < 1e-12                  # tail-sum identity (Eq. 2)
    if 0 < b < 1:                                        # Pr(L >= j) = beta^j
        np.testing.assert_allclose(tail, [b ** j for j in range(1, d + 1)], rtol=1e-6)


def test_tail_probabilities_are_products_of_beta():
    """P6/P7 for general independent rows: averaging the exact outcome over draft paths
    x_j ~ q_j gives Pr(L >= j) = prod_{i<j} beta_i with beta_i = 1 - TV (scipy)."""
    rng = np.random.default_rng(7)
    V, k = 12, 3
    zp = rng.normal(0, 1.5, (k + 1, V)).astype(np.float32)
    zq = rng.normal(0, 1.5, (k, V)).astype(np.float32)
    paths = np.array(list(itertools.product(range(V), repeat=k)), np.int32)
    n = len(paths)
    out = oracle.outcome_dist(np.broadcast_to(zp, (n, k + 1, V)).copy(),
                              np.broadcast_to(zq, (n, k, V)).copy(), paths, 1.0)
    qs = sm(zq)
    w = np.prod([qs[j][paths[:, j]] for j in range(k)], axis=0)
    pL = (w[:, None] * out.sum(-1)).sum(0)
    beta = [1 - 0.5 * np.abs(sm(zp[j]) - qs[j]).sum() for j in range(k)]
    for j in range(1, k + 1):
        assert abs(pL[j:].sum() - np.prod(beta[:j])) < 1e-12


def test_residual_mass_is_one_minus_beta():
    """P3: at a rejection, R = sum_x max(0, p-q) = 1 - sum_x min(p,q)."""
    d = make_batch(V=300, k=4, B=200, T=1.0, kappa=30.0, seed=11)
    L, tok, st, tr = oracle.verify(d["p"], d["q"], d["ids"], 1.0, seed=3, trace=True)
    n = 0
    for b in range(200):
        if L[b] < 4:
            j = L[b]
            beta = 1 - 0.5 * np.abs(sm(d["p"][b, j]) - sm(d["q"][b, j])).sum()
            assert abs(tr[b].R - (1 - beta)) < 1e-12
            n += 1
    assert n > 50


def test_inverse_cdf_hand_worked():
    """tests/golden inverse_cdf_hand: decisions and tokens follow the hand-derived rule."""
    ex = WORKED["inverse_cdf_hand"]
    B = 4000
    p = np.broadcast_to(np.stack([logits(ex["p0"]), logits(ex["p1"])]), (B, 2, 4)).copy()
    q = np.broadcast_to(logits(ex["q0"])[None], (B, 1, 4)).copy()
    ids = np.zeros((B, 1), np.int32)
    L, tok, st = oracle.verify(p, q, ids, 1.0, seed=42, round=5, rid_base=0)
    checked = 0
    for b in range(B):
        ua, _ = oracle.uniforms(42, 0, 5, b)
        if abs(ua - ex["a0"]) < 1e-6:
            continue
        if ua >= ex["a0"]:
            _, us = oracle.uniforms(42, 0, 5, b)
            th = us * ex["R"]
            if abs(th - 0.1) < 1e-6:
                continue
            assert L[b] == 0 and tok[b, 0] == (2 if th < 0.1 else 3)
        else:
            _, us = oracle.uniforms(42, 1, 5, b)
            cdf = np.array(ex["bonus_cdf"])
            if np.min(np.abs(cdf - us)) < 1e-6:
                continue
            assert L[b] == 1 and tok[b, 0] == 0 and tok[b, 1] == int(np.argmax(cdf > us))
        checked += 1
    assert checked > 3900
    assert 0.2 < np.mean(L == 1) < 0.3


# ---------------------------------------------------------------- special cases (P8) --------
def test_identical_rows_accept_everything():
    d = make_batch(V=500, k=5, B=300, T=1.0, kappa=30.0, seed=12)
    q = d["p"][:, :5].copy()
    rng = np.random.default_rng(0)
    ids = np.stack([[rng.choice(500, p=sm(q[b, j])) for j in range(5)] for b in range(300)])
    L, tok, st = oracle.verify(d["p"], q, ids.astype(np.int32), 1.0, seed=1)
    assert np.all(L == 5) and np.all(st == 0)
    np.testing.assert_array_equal(tok[:, :5], ids)


def test_disjoint_one_hots_reject_with_target_token():
    V, k = 10, 3
    p = np.full((1, k + 1, V), -np.inf, np.float32)
    q = np.full((1, k, V), -np.inf, np.float32)
    p[0, :, 7] = 0.0
    q[0, :, 2] = 0.0
    for seed in range(50):
        L, tok, st = oracle.verify(p, q, np.full((1, k), 2, np.int32), 1.0, seed=seed)
        assert L[0] == 0 and tok[0, 0] == 7 and list(tok[0, 1:]) == [-1] * k
        assert st[0] == 0


def test_k1_is_single_token_leviathan_sampling():
    """k = 1 and x ~ q: first token ~ p_0 (single-step speculative sampling)."""
    rng = np.random.default_rng(8)
    V, B = 7, 60000
    zp = rng.normal(0, 1, (2, V)).astype(np.float32)
    zq = rng.normal(0, 1, (1, V)).astype(np.float32)
    ids = rng.choice(V, B, p=sm(zq[0]))[:, None].astype(np.int32)
    L, tok, _ = oracle.verify(np.broadcast_to(zp, (B, 2, V)).copy(),
                              np.broadcast_to(zq, (B, 1, V)).copy(), ids, 1.0, seed=4,
                              n_threads=4)
    obs = np.bincount(tok[:, 0], minlength=V)
    exp = B * sm(zp[0])
    assert stats.chi2.sf(((obs - exp) ** 2 / exp).sum(), V - 1) > 1e-4
    # conditional on full acceptance the bonus follows p_1 (P8 v)
    acc = L == 1
    obs = np.bincount(tok[acc, 1], minlength=V)
    exp = acc.sum() * sm(zp[1])
    assert stats.chi2.sf(((obs - exp) ** 2 / exp).sum(), V - 1) > 1e-4


# ---------------------------------------------------------------- greedy (P9) ---------------
def test_greedy_matches_torch_argmax():
    import torch
    rng = np.random.default_rng(9)
    B, k, V = 400, 4, 64
    p = rng.integers(-3, 3, (B, k + 1, V)).astype(np.float32)   # many ties
    g = torch.argmax(torch.from_numpy(p), dim=-1).numpy()        # first index on ties
    ids = g[:, :k].copy().astype(np.int32)
    flip = rng.random((B, k)) < 0.25
    ids[flip] = (ids[flip] + 1) % V
    L, tok, st = oracle.verify(p, None, ids, 0.0)
    for b in range(B):
        mism = np.nonzero(ids[b] != g[b, :k])[0]
        Lb = mism[0] if len(mism) else k
        assert L[b] == Lb
        assert list(tok[b, :Lb]) == list(ids[b, :Lb]) and tok[b, Lb] == g[b, Lb]
        assert np.all(tok[b, Lb + 1:] == -1)


# ---------------------------------------------------------------- faults & input forms -----
def test_faults_and_laziness():
    d = make_batch(V=100, k=3, B=4, T=1.0, kappa=30.0, seed=13)
    p, q, ids = d["p"].copy(), d["q"].copy(), d["ids"].copy()
    # request 0: NaN in p_0 -> hard fault
    p[0, 0, 5] = np.nan
    # request 1: bad draft id at position 0
    ids[1, 0] = 100
    # request 2: force rejection at 0 (draft token impossible under p), NaN in p_2: never read
    p[2, 0, ids[2, 0]] = -np.inf
    p[2, 2, 7] = np.nan
    # request 3: all -inf q_0 row -> empty-row fault
    q[3, 0, :] = -np.inf
    L, tok, st = oracle.verify(p, q, ids, 1.0, seed=1)
    assert st[0] == oracle.FAULT_NONFINITE and L[0] == 0 and np.all(tok[0] == -1)
    assert st[1] == oracle.FAULT_BAD_DRAFT_ID and np.all(tok[1] == -1)
    assert st[2] == 0 and L[2] == 0 and tok[2, 0] >= 0
    assert st[3] == oracle.FAULT_EMPTY_ROW and np.all(tok[3] == -1)


def test_zero_q_is_a_rejection():
    d = make_batch(V=50, k=2, B=1, T=1.0, kappa=30.0, seed=14)
    q = d["q"].copy()
    q[0, 0, d["ids"][0, 0]] = -np.inf
    L, tok, st = oracle.verify(d["p"], q, d["ids"], 1.0, seed=2)
    assert L[0] == 0 and st[0] == oracle.FAULT_ZERO_Q and tok[0, 0] >= 0


def test_bf16_and_padding_are_exact_widenings():
    d = make_batch(V=333, k=3, B=40, T=1.0, kappa=10.0, seed=15, dtype="bf16")
    L, tok, st = oracle.verify(d["p"], d["q"], d["ids"], 1.0, seed=5)
    pf = (d["p"].astype(np.uint32) << 16).view(np.float32)
    qf = (d["q"].astype(np.uint32) << 16).view(np.float32)
    L2, tok2, _ = oracle.verify(pf, qf, d["ids"], 1.0, seed=5)
    np.testing.assert_array_equal(L, L2)
    np.testing.assert_array_equal(tok, tok2)
    dp = make_batch(V=333, k=3, B=40, T=1.0, kappa=10.0, seed=15, ld=344)
    dc = make_batch(V=333, k=3, B=40, T=1.0, kappa=10.0, seed=15)
    L3, tok3, st3 = oracle.verify(dp["p"], dp["q"], dp["ids"], 1.0, seed=5, V=333)
    L4, tok4, _ = oracle.verify(dc["p"], dc["q"], dc["ids"], 1.0, seed=5)
    assert np.all(st3 == 0)
    np.testing.assert_array_equal(L3, L4)
    np.testing.assert_array_equal(tok3, tok4)
    assert np.array_equal(bf16_bits(np.array([1.0], np.float32)), np.array([0x3F80], np.uint16))


def test_threads_do_not_change_results():
    d = make_batch(V=1000, k=4, B=64, T=1.0, kappa=30.0, seed=16)
    a = oracle.verify(d["p"], d["q"], d["ids"], 1.0, seed=8, n_threads=1)
    b = oracle.verify(d["p"], d["q"], d["ids"], 1.0, seed=8, n_threads=7)
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x, y)
