"""Pins of the tree-verification oracle (reading D-2): recursive rejection
sampling over the i.i.d. children of each node of a full m-ary tree.

* m = 1 is the chain: identical results to sd_ref_verify (itself pinned) on the same rows;
* losslessness by exact enumeration: over every tree whose children are drawn i.i.d. from their
  parent's q (prefix-conditioned tables, V = 3, m = 2, d = 2 and V = 4, m = 3, d = 1), the emitted
  sequence completed by target sampling is distributed exactly as the target's autoregressive
  joint (TV <= 1e-12) -- the property the paper's best-of-paths rule lacks;
* the step-by-step walk against the exact outcome distribution (Monte Carlo, G-test);
* greedy trees follow numpy's argmax.
"""
import itertools

import numpy as np
import pytest
from scipy import stats

import oracle
from workload import make_batch, make_tiny_tables


def tree_from_tables(P, Q, m, d, cand):
    """Rows of a full m-ary tree whose non-root nodes carry the tokens `cand` (level order)."""
    N, Nint = oracle.tree_nodes(m, d)
    tok = np.zeros(N, np.int32)
    tok[1:] = cand
    pre = [()] * N
    for n in range(1, N):
        pre[n] = pre[(n - 1) // m] + (int(tok[n]),)
    p = np.stack([P[pre[n]] for n in range(N)])
    q = np.stack([Q[pre[n]] for n in range(Nint)])
    return p, q, tok, pre


def test_m1_tree_is_the_chain():
    d = make_batch(V=200, k=4, B=300, T=1.0, kappa=10.0, seed=5)
    B, k = d["ids"].shape
    tok = np.zeros((B, k + 1), np.int32)
    tok[:, 1:] = d["ids"]
    for T in (1.0, 0.0):
        L, toks, st, node, mu = oracle.tree_verify(d["p"], d["q"] if T else None, tok, 1, k, T,
                                                   seed=9, round=3, rid_base=70)
        rL, rtok, rst = oracle.verify(d["p"], d["q"] if T else None, d["ids"], T, seed=9, round=3,
                                      rid_base=70)
        np.testing.assert_array_equal(L, rL)
        np.testing.assert_array_equal(toks, rtok)
        np.testing.assert_array_equal(st, rst)


@pytest.mark.parametrize("V,m,d", [(3, 2, 2), (4, 3, 1)])
def test_lossless_by_exact_enumeration(V, m, d):
    P, Q = make_tiny_tables(V=V, k=d, seed=77 + V, alpha=1.0)
    sm = lambda z: np.exp(z.astype(np.float64) - np.logaddexp.reduce(z.astype(np.float64)))  # noqa: E731
    N, Nint = oracle.tree_nodes(m, d)
    joint = {}
    total_w = 0.0
    for cand in itertools.product(range(V), repeat=N - 1):
        p, q, tok, pre = tree_from_tables(P, Q, m, d, np.array(cand, np.int32))
        w = 1.0
        for n in range(1, N):                        # children ~ q of their parent, i.i.d.
            w *= sm(Q[pre[(n - 1) // m]])[cand[n - 1]]
        total_w += w
        out = oracle.tree_outcome_dist(p[None], q[None], tok[None], m, d, 1.0)[0]
        for n in range(N):
            for y in range(V):
                pr = out[n, y]
                if pr == 0.0:
                    continue
                s0 = pre[n] + (y,)
                # complete the emitted prefix with target sampling to d + 1 tokens
                stack = [(s0, w * pr)]
                while stack:
                    s, ps = stack.pop()
                    if len(s) == d + 1:
                        joint[s] = joint.get(s, 0.0) + ps
                        continue
                    nxt = sm(P[s])
                    for z in range(V):
                        stack.append((s + (z,), ps * nxt[z]))
    assert abs(total_w - 1.0) < 1e-12
    tv = 0.0
    for s in itertools.product(range(V), repeat=d + 1):
        target = 1.0
        for t in range(d + 1):
            target *= sm(P[s[:t]])[s[t]]
        tv += abs(joint.get(s, 0.0) - target)
    assert 0.5 * tv < 1e-12, tv


def test_walk_matches_the_exact_outcome_distribution():
    """One fixed tree (V = 6, m = 2, d = 2), 40000 walks with fresh uniforms (request ids):
    the stop-node x emitted-token frequencies follow sd_ref_tree_outcome_dist (G-test)."""
    P, Q = make_tiny_tables(V=6, k=2, seed=31, alpha=0.7)
    rng = np.random.default_rng(2)
    p, q, tok, pre = tree_from_tables(P, Q, 2, 2, rng.integers(0, 6, 6).astype(np.int32))
    R = 40000
    L, toks, st, node, mu = oracle.tree_verify(np.broadcast_to(p, (R,) + p.shape).copy(),
                                               np.broadcast_to(q, (R,) + q.shape).copy(),
                                               np.broadcast_to(tok, (R, tok.size)).copy(),
                                               2, 2, 1.0, seed=4, round=0, rid_base=0)
    exact = oracle.tree_outcome_dist(p[None], q[None], tok[None], 2, 2, 1.0)[0]
    emitted = toks[np.arange(R), L]
    obs = np.zeros_like(exact)
    np.add.at(obs, (node, emitted), 1)
    keep = exact * R > 5
    g = 2 * np.sum(obs[keep] * np.log(np.maximum(obs[keep], 1) / (R * exact[keep])))
    assert stats.chi2.sf(g, keep.sum() - 1) > 1e-4
    assert obs[~keep].sum() <= 5 * max(1, (~keep).sum())
    assert abs(exact.sum() - 1.0) < 1e-12


def test_greedy_tree_follows_argmax():
    P, Q = make_tiny_tables(V=5, k=3, seed=3, alpha=1.0)
    rng = np.random.default_rng(4)
    m, d = 2, 3
    for _ in range(50):
        p, q, tok, pre = tree_from_tables(P, Q, m, d, rng.integers(0, 5, oracle.tree_nodes(m, d)[0] - 1).astype(np.int32))
        L, toks, st, node, mu = oracle.tree_verify(p[None], None, tok[None], m, d, 0.0)
        n, path = 0, []
        for t in range(d + 1):
            g = int(np.argmax(p[n]))
            kids = [m * n + 1 + i for i in range(m)] if t < d else []
            nxt = next((c for c in kids if tok[c] == g), None)
            path.append(g)
            if nxt is None:
                break
            n = nxt
        assert L[0] == len(path) - 1 and list(toks[0, :len(path)]) == path


def test_candidate_uniform_counters():
    """Hand examples fixing the uniforms' counters (reading D-2), root with m = 2 children, d = 1.
    (a) p = [.25, .25, .5], q = [.5, .5, 0], candidates (token 0, token 1): a_0 = .5 is decided by
        u24(w0) of counter (0, round, rid); after a rejection d_1 = norm(max(0, p - q)) = [0, 0, 1],
        so token 1 has a_1 = 0 and token 2 is emitted.
    (b) p = [0, .35, .65], q = [.4, .3, .3], candidates (0, 1): token 0 has p = 0 (rejected);
        d_1 = [0, .05, .35] / .4 = [0, .125, .875], so token 1 passes with a_1 = .125/.3 = 5/12,
        decided by u24(w0) of counter (0 + 32 * 1, round, rid); otherwise d_2 = [0, 0, 1] emits 2."""
    lg = lambda v: np.log(np.asarray(v, np.float64)).astype(np.float32)  # noqa: E731
    m, d, B = 2, 1, 2000
    leaf = lg([1 / 3] * 3)
    tok = np.array([0, 0, 1], np.int32)

    def run(prow, qrow):
        p = np.stack([lg(prow), leaf, leaf])
        q = lg(qrow)[None]
        return oracle.tree_verify(np.broadcast_to(p, (B, 3, 3)).copy(),
                                  np.broadcast_to(q, (B, 1, 3)).copy(),
                                  np.broadcast_to(tok, (B, 3)).copy(), m, d, 1.0, seed=6, round=2,
                                  rid_base=0)

    L, toks, _, _, _ = run([.25, .25, .5], [.5, .5, 1e-30])
    L4, toks4, _, _, _ = run([1e-30, .35, .65], [.4, .3, .3])
    for b in range(B):
        u0, _ = oracle.uniforms(6, 0, 2, b)
        u1, _ = oracle.uniforms(6, 32, 2, b)
        if abs(u0 - 0.5) > 1e-6:
            assert (L[b], toks[b, 0]) == ((1, 0) if u0 < 0.5 else (0, 2))
        if abs(u1 - 5 / 12) > 1e-6:
            assert (L4[b], toks4[b, 0]) == ((1, 1) if u1 < 5 / 12 else (0, 2))
