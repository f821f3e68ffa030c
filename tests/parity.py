"""The C-13 parity rule: compare a GPU verify result with the oracle.

1. greedy: exact equality always.
2. sampled, request not a tie: L, tokens and status bit-identical.
   A request is a tie when the oracle's fp64 margins are below tau = 1e-6:
   min |u_acc(j) - a_j| over the tests it decided, the inverse-CDF margin
   min(theta - C(t-1), C(t) - theta) / R, or R < 5e-8.
3. tie: the GPU result must be consistent with the oracle's fp64 quantities within tau: every
   acceptance decision the GPU implies (accept j < L_gpu, reject at L_gpu) agrees with the
   oracle's a_j wherever |u - a_j| >= tau, and its token t' satisfies
   C(t'-1) - tau R <= theta <= C(t') + tau R at the GPU's L.
4. tie budget: callers assert the tie fraction they expect.
"""
from __future__ import annotations

import numpy as np

import oracle

TAU = 1e-6
R_MIN = 5e-8


def compare(inp, gpu, ref, T, seed, round=0, rid_base=0, V=None):
    """inp: dict(p, q, ids) numpy; gpu/ref: (L, tok, status[, trace]).  Returns stats dict;
    raises AssertionError with the first violating request."""
    gL, gtok, gst = [np.asarray(x) for x in gpu[:3]]
    rL, rtok, rst, tr = ref
    B, k = inp["ids"].shape
    ties = 0
    for b in range(B):
        hard = rst[b] & oracle.HARD_FAULTS
        exact = T == 0.0 or hard
        if not exact:
            t = tr[b]
            tie = t.mu_a < TAU or t.mu_s < TAU or t.R < R_MIN
            exact = not tie
        if exact:
            assert gL[b] == rL[b] and np.array_equal(gtok[b], rtok[b]) and gst[b] == rst[b], (
                f"request {b}: gpu L={gL[b]} tok={gtok[b].tolist()} st={gst[b]} vs oracle "
                f"L={rL[b]} tok={rtok[b].tolist()} st={rst[b]}")
            continue
        ties += 1
        _check_tie(inp, b, int(gL[b]), gtok[b], T, seed, round, rid_base, V)
    return {"ties": ties, "n": B}


def _check_tie(inp, b, Lg, tokg, T, seed, round, rid_base, V):
    p, q, ids = inp["p"], inp["q"], inp["ids"]
    k = ids.shape[1]
    a, u = oracle.accept_probs(p, q, ids, b, T, seed, round, rid_base, V=V)
    for j in range(Lg + (0 if Lg == k else 1)):
        gpu_accepts = j < Lg
        ref_accepts = u[j] < a[j] or a[j] >= 1.0
        if gpu_accepts != ref_accepts:
            assert abs(u[j] - a[j]) < TAU, f"request {b} position {j}: decision differs, " \
                                           f"|u-a|={abs(u[j] - a[j])}"
    assert np.array_equal(tokg[:Lg], ids[b, :Lg]), f"request {b}: accepted prefix differs"
    assert np.all(tokg[Lg + 1:] == -1)
    t = int(tokg[Lg])
    Cp, Ct, R, th = oracle.sample_check(p, q, ids, b, Lg, t, T, seed, round, rid_base, V=V)
    assert Cp - TAU * R <= th <= Ct + TAU * R, (
        f"request {b}: token {t} outside its CDF cell: C(t-1)={Cp} theta={th} C(t)={Ct} R={R}")
