"""GPU parity of the lossless tree verification (sd_tree_verify) against the
tree oracle (tests/test_oracle_tree.py pins it): bit-exact accept lengths, tokens, stop nodes and
status outside decision ties (oracle margin < 1e-6), greedy trees exactly, and the GPU's walk
distribution against the exact outcome distribution (G-test)."""
import os

import numpy as np
import pytest
import torch
from scipy import stats

import oracle
from workload import make_batch, make_tiny_tables

pytestmark = pytest.mark.gpu

sd = pytest.importorskip("paper_2601_21622_b200")
DEV = torch.device("cuda:0")
TAU = 1e-6


def _dev(a):
    t = torch.from_numpy(np.ascontiguousarray(a))
    if a.dtype == np.uint16:
        t = t.view(torch.bfloat16)
    return t.to(DEV)


def tree_batch(V, m, d, B, T, seed, dtype="f32"):
    """Rows of B full m-ary trees: LLM-like target rows at every node, draft rows at internal
    nodes, each child's token drawn from its parent's draft distribution (Gumbel-max)."""
    N, Nint = oracle.tree_nodes(m, d)
    b = make_batch(V=V, k=N - 1, B=B, T=max(T, 1e-3), kappa=30.0, seed=seed, dtype=dtype)
    p, q = b["p"], b["q"][:, :Nint]
    qf = (q.astype(np.uint32) << 16).view(np.float32) if dtype == "bf16" else q
    rng = np.random.default_rng(seed + 1)
    tok = np.zeros((B, N), np.int32)
    for n in range(Nint):
        z = qf[:, n].astype(np.float64) / max(T, 1e-3)
        for i in range(m):
            g = -np.log(-np.log(rng.random(z.shape)))
            tok[:, m * n + 1 + i] = np.argmax(z + g, axis=-1) if T > 0 else np.argmax(z, axis=-1)
    return p, np.ascontiguousarray(q), tok


@pytest.mark.parametrize("V,m,d,B,T,dtype", [(32000, 2, 3, 48, 1.0, "f32"), (32000, 3, 2, 48, 0.7, "f32"),
                                             (32000, 2, 3, 32, 1.0, "bf16"), (4100, 1, 5, 64, 1.0, "f32"),
                                             (32000, 2, 3, 48, 0.0, "f32"), (128256, 2, 2, 8, 1.0, "f32")])
def test_tree_verify_matches_the_oracle(V, m, d, B, T, dtype):
    per16 = 4 if dtype == "f32" else 8
    if V % per16:
        pytest.skip("rows must be 16-byte multiples")
    p, q, tok = tree_batch(V, m, d, B, T, seed=V + 10 * m + d, dtype=dtype)
    L, toks, st, node = sd.tree_verify(_dev(p), _dev(q) if T > 0 else None, _dev(tok), m, T,
                                       seed=3, round=4, request_id_base=100)
    torch.cuda.synchronize()
    L, toks, st, node = (x.cpu().numpy() for x in (L, toks, st, node))
    rL, rtoks, rst, rnode, rmu = oracle.tree_verify(p, q if T > 0 else None, tok, m, d, T, seed=3,
                                                    round=4, rid_base=100)
    tie = (rmu < TAU) if T > 0 else np.zeros(B, bool)
    ok = ~tie
    np.testing.assert_array_equal(L[ok], rL[ok])
    np.testing.assert_array_equal(toks[ok], rtoks[ok])
    np.testing.assert_array_equal(node[ok], rnode[ok])
    np.testing.assert_array_equal(st[ok], rst[ok])
    assert tie.mean() <= 0.05
    if T > 0:
        assert L.mean() > 0.3                    # the trees do accept tokens


def test_tree_walk_distribution_matches_the_exact_outcome():
    """One fixed tree (V = 8, m = 2, d = 2) walked by 20000 GPU requests with distinct Philox
    streams: the (stop node, emitted token) frequencies follow sd_ref_tree_outcome_dist."""
    P, Q = make_tiny_tables(V=8, k=2, seed=91, alpha=0.8)
    m, d = 2, 2
    N, Nint = oracle.tree_nodes(m, d)
    rng = np.random.default_rng(5)
    cand = rng.integers(0, 8, N - 1).astype(np.int32)
    tok = np.zeros(N, np.int32)
    tok[1:] = cand
    pre = [()] * N
    for n in range(1, N):
        pre[n] = pre[(n - 1) // m] + (int(tok[n]),)
    p = np.stack([P[pre[n]] for n in range(N)])
    q = np.stack([Q[pre[n]] for n in range(Nint)])
    R = 20000
    L, toks, st, node = sd.tree_verify(_dev(np.broadcast_to(p, (R, N, 8)).copy()),
                                       _dev(np.broadcast_to(q, (R, Nint, 8)).copy()),
                                       _dev(np.broadcast_to(tok, (R, N)).copy()), m, 1.0, seed=8)
    torch.cuda.synchronize()
    L, toks, node = L.cpu().numpy(), toks.cpu().numpy(), node.cpu().numpy()
    exact = oracle.tree_outcome_dist(p[None], q[None], tok[None], m, d, 1.0)[0]
    obs = np.zeros_like(exact)
    np.add.at(obs, (node, toks[np.arange(R), L]), 1)
    keep = exact * R > 5
    g = 2 * np.sum(obs[keep] * np.log(np.maximum(obs[keep], 1) / (R * exact[keep])))
    assert stats.chi2.sf(g, keep.sum() - 1) > 1e-4


def test_tree_verify_one_cta_kernel_matches_the_oracle():
    """STARSD_TREE_CLUSTER=0 -- the one-CTA-per-request tree kernel instead of the 8-CTA cluster
    (the knob is read once per process, so in a subprocess): the same parity cases as above."""
    if os.environ.get("STARSD_TREE_CLUSTER") == "0":
        pytest.skip("(running inside the subprocess)")
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider", "-m", "gpu",
                        os.path.abspath(__file__), "-k", "matches_the_oracle and not one_cta"],
                       env=dict(os.environ, STARSD_TREE_CLUSTER="0"), capture_output=True, text=True,
                       timeout=900, cwd=root)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert "6 passed" in r.stdout, r.stdout[-1000:]
