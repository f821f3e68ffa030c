"""GPU checks of the draft side and the exchange-minimal verify:

* sd_draft_sample against the oracle's draft sampler (tests/test_oracle_checkers.py pins it):
  tokens identical outside CDF-cell ties (margin < 1e-6), log q(x) within 1e-5;
* sd_verify_qmeta (draft rows as metadata, q rows read only at the stop position) against
  sd_verify on the same rows: bit-identical accept lengths, tokens and status -- also when every
  q row except the stop rows is poisoned with NaN (it is never read) -- and against the oracle;
* the draft -> verify chain end to end: draft-sampled tokens verified lazily follow the oracle.
"""
import os

import numpy as np
import pytest
import torch

import oracle
from parity import compare
from workload import CONFIGS, make_batch, make_batch_torch

pytestmark = pytest.mark.gpu

sd = pytest.importorskip("paper_2601_21622_b200")
DEV = torch.device("cuda:0")
NTH = max(1, len(os.sched_getaffinity(0)))


def _host(t):
    if t.dtype == torch.bfloat16:
        return t.view(torch.int16).cpu().numpy().view(np.uint16)
    return t.cpu().numpy()


def _dev(a):
    t = torch.from_numpy(np.ascontiguousarray(a))
    if a.dtype == np.uint16:
        t = t.view(torch.bfloat16)
    return t.to(DEV)


@pytest.mark.parametrize("V,k,B,T,dtype", [(32000, 5, 64, 1.0, "f32"), (32000, 5, 64, 0.7, "bf16"),
                                           (128256, 7, 16, 1.0, "f32"), (1003, 3, 50, 1.0, "f32"),
                                           (32000, 5, 64, 0.0, "f32"), (300000, 2, 4, 1.0, "f32")])
def test_draft_sampler_matches_the_oracle(V, k, B, T, dtype):
    per16 = 4 if dtype == "f32" else 8
    ld = (V + per16 - 1) // per16 * per16                # rows padded to 16 bytes (NaN padding)
    d = make_batch(V=V, k=k, B=B, T=max(T, 1e-3), kappa=30.0, seed=V + B, dtype=dtype, ld=ld)
    q = _dev(d["q"])
    ids, qm, st = sd.draft_sample(q, T, seed=17, round=3, request_id_base=900, vocab=V)
    torch.cuda.synchronize()
    ids = ids.cpu().numpy()
    rid, rlogq, rmu, rst = oracle.draft_sample(d["q"], T, seed=17, round=3, rid_base=900, V=V)
    tie = rmu < 1e-6
    assert np.array_equal(ids[~tie], rid[~tie]), np.argwhere(ids != rid)[:5]
    assert tie.mean() <= 1e-2
    np.testing.assert_array_equal(st.cpu().numpy(), rst)
    if T > 0:
        f = sd.qmeta_fields(qm)
        c2 = np.float32(1.4426950408889634 / T)
        logq = np.log(2.0) * (f["zx"].double().cpu().numpy() * np.float64(c2)
                              - f["D"].double().cpu().numpy() - np.log2(f["S"].cpu().numpy()))
        ok = ~tie
        assert np.max(np.abs(logq[ok] - rlogq[ok])) < 1e-5


@pytest.mark.parametrize("cfg,dtype", [("c2", "f32"), ("c3", "f32"), ("c2", "bf16"), ("c3", "bf16")])
def test_lazy_q_verify_is_bit_identical_to_full_verify(cfg, dtype):
    c = CONFIGS[cfg]
    B = c["B"] if cfg == "c2" else 64
    t = make_batch_torch(V=c["V"], k=c["k"], B=B, T=1.0, kappa=c["kappa"], seed=c["seed"] + 3,
                         device=DEV, dtype=dtype)
    qm = sd.draft_qmeta(t["q"], t["ids"], 1.0)
    full = sd.verify(t["p"], t["q"], t["ids"], 1.0, seed=8, round=2, request_id_base=64)
    lazy = sd.verify_qmeta(t["p"], t["q"], qm, t["ids"], 1.0, seed=8, round=2, request_id_base=64)
    torch.cuda.synchronize()
    for a, b in zip(full, lazy):
        assert torch.equal(a, b)
    # q rows other than each request's stop row are never read: poison them
    L = full[0].long()
    poison = torch.full_like(t["q"], float("nan"))
    rows = torch.nonzero(L < c["k"]).squeeze(1)
    poison[rows, L[rows]] = t["q"][rows, L[rows]]
    lazy2 = sd.verify_qmeta(t["p"], poison, qm, t["ids"], 1.0, seed=8, round=2, request_id_base=64)
    torch.cuda.synchronize()
    for a, b in zip(full, lazy2):
        assert torch.equal(a, b)
    d = {x: _host(t[x]) for x in ("p", "q", "ids")}
    ref = oracle.verify(d["p"], d["q"], d["ids"], 1.0, seed=8, round=2, rid_base=64, trace=True,
                        n_threads=NTH)
    compare(d, tuple(x.cpu().numpy() for x in lazy), ref, 1.0, 8, 2, 64)


def test_lazy_q_verify_faults_and_zero_q():
    """Fault bits travel in the metadata: a NaN q row and an all -inf q row at position 0 are hard
    faults, a draft token with q(x) = 0 is the C-7 rejection -- exactly as in sd_verify."""
    d = make_batch(V=4096, k=3, B=6, T=1.0, kappa=30.0, seed=12)
    d["q"][0, 0, 5] = np.nan
    d["q"][1, 0, :] = -np.inf
    d["q"][2, 0, d["ids"][2, 0]] = -np.inf
    p, q, ids = _dev(d["p"]), _dev(d["q"]), _dev(d["ids"])
    qm = sd.draft_qmeta(q, ids, 1.0)
    full = sd.verify(p, q, ids, 1.0, seed=1)
    lazy = sd.verify_qmeta(p, q, qm, ids, 1.0, seed=1)
    torch.cuda.synchronize()
    for a, b in zip(full, lazy):
        assert torch.equal(a, b)
    st = lazy[2].cpu().numpy()
    assert st[0] == sd.FAULT_NONFINITE and st[1] == sd.FAULT_EMPTY_ROW and st[2] & sd.FAULT_ZERO_Q


def test_draft_then_lazy_verify_chain_follows_the_oracle():
    """Draft-sampled tokens (NEXT-2) verified with their metadata (NEXT-1) -- the star's
    exchange-minimal round -- match the oracle run on the same rows and tokens."""
    c = CONFIGS["c3"]
    t = make_batch_torch(V=c["V"], k=c["k"], B=32, T=1.0, kappa=c["kappa"], seed=c["seed"] + 11,
                         device=DEV)
    ids, qm, st = sd.draft_sample(t["q"], 1.0, seed=4, round=7, request_id_base=32)
    assert int((st != 0).sum()) == 0
    L, tok, vst = sd.verify_qmeta(t["p"], t["q"], qm, ids, 1.0, seed=4, round=7, request_id_base=32)
    torch.cuda.synchronize()
    d = {"p": _host(t["p"]), "q": _host(t["q"]), "ids": ids.cpu().numpy()}
    ref = oracle.verify(d["p"], d["q"], d["ids"], 1.0, seed=4, round=7, rid_base=32, trace=True,
                        n_threads=NTH)
    compare(d, (L.cpu().numpy(), tok.cpu().numpy(), vst.cpu().numpy()), ref, 1.0, 4, 7, 32)
    rid = oracle.draft_sample(d["q"], 1.0, seed=4, round=7, rid_base=32)
    tie = rid[2] < 1e-6
    assert np.array_equal(d["ids"][~tie], rid[0][~tie])
