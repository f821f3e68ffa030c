"""Star exchange + round scheduler on one GPU through the C ABI, using the
loopback transport: one process plays the draft and N virtual verifiers, the exchange is a
device copy on each pair's stream, and every round's results are checked against the oracle
(DESIGN.md "Parity").  The NCCL transport shares the scheduler, poll and stats code; it needs
two GPUs and is exercised by tools/star_demo.py under torchrun."""
import numpy as np
import pytest
import torch

import oracle
from parity import compare
from workload import make_batch

pytestmark = pytest.mark.gpu

star = pytest.importorskip("paper_2601_21622_b200.star")
DEV = torch.device("cuda:0")


def _dev(a):
    return None if a is None else torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


@pytest.mark.parametrize("T,payload", [(1.0, "full"), (0.0, "full"), (1.0, "qmeta")])
def test_loopback_rounds_match_oracle_in_fifo_order(T, payload):
    """payload="qmeta" (NEXT-1): only ids + 24-byte metadata per draft token go out; the virtual
    verifier reads its stop rows from the draft's q rows (sd_verify_qmeta)."""
    import paper_2601_21622_b200 as sd
    N, slots, rounds_per_stream, B, k, V = 3, 2, 4, 24, 4, 3000
    seed = 77
    h = star.Star(0, N + 1, B, k, V, T, seed=seed, n_slots=slots, device=DEV, transport="loopback",
                  payload=payload)
    inflight, done = {}, []

    def submit(v, s, r):
        d = make_batch(V, k, B, T, 30.0, seed=1000 * v + 10 * s + r)
        t = {"p": _dev(d["p"]), "q": _dev(d["q"]) if T > 0 else None, "ids": _dev(d["ids"]),
             "L": torch.full((B,), -7, dtype=torch.int32, device=DEV),
             "tok": torch.full((B, k + 1), -7, dtype=torch.int32, device=DEV)}
        rid = (v << 40) + (s << 20)
        qm = sd.draft_qmeta(t["q"], t["ids"], T) if payload == "qmeta" else None
        t["qm"] = qm
        h.submit(v, s, r, t["ids"], t["q"], t["L"], t["tok"], request_id_base=rid, p=t["p"],
                 qmeta=qm)
        inflight[(v, s)] = (r, d, t, rid)

    for s in range(slots):
        for v in range(1, N + 1):
            submit(v, s, 0)
    while inflight:
        got = h.poll(timeout_us=10_000_000)
        assert got is not None, "no return within 10 s"
        v, s, r = got
        r0, d, t, rid = inflight.pop((v, s))
        assert r == r0
        L, tok = t["L"].cpu().numpy(), t["tok"].cpu().numpy()
        ref = oracle.verify(d["p"], d["q"] if T > 0 else None, d["ids"], T, seed=seed, round=r,
                            rid_base=rid, trace=True)
        compare(d, (L, tok, np.zeros(B, np.int32)), ref, T, seed, r, rid)
        done.append((v, s, r))
        if r + 1 < rounds_per_stream:
            h.draft_begin()
            submit(v, s, r + 1)
            h.draft_end()
    assert sorted(done) == sorted((v, s, r) for v in range(1, N + 1) for s in range(slots)
                                  for r in range(rounds_per_stream))
    st = h.stats()
    assert st["rounds"] == N * slots * rounds_per_stream
    assert 0.0 < st["busy_fraction"] <= 1.0 + 1e-9
    assert st["mean_wait_ms"] >= 0.0
    h.close()


def test_loopback_rejects_misuse():
    h = star.Star(0, 2, 8, 2, 64, 1.0, n_slots=1, device=DEV, transport="loopback")
    ids = torch.zeros(8, 2, dtype=torch.int32, device=DEV)
    q = torch.zeros(8, 2, 64, device=DEV)
    p = torch.zeros(8, 3, 64, device=DEV)
    L = torch.empty(8, dtype=torch.int32, device=DEV)
    tok = torch.empty(8, 3, dtype=torch.int32, device=DEV)
    with pytest.raises(star.StarsdError, match="INVALID_ARGUMENT"):
        h.submit(2, 0, 0, ids, q, L, tok, p=p)          # verifier out of range
    with pytest.raises(star.StarsdError, match="INVALID_ARGUMENT"):
        h.submit(1, 1, 0, ids, q, L, tok, p=p)          # slot out of range
    h.submit(1, 0, 0, ids, q, L, tok, p=p)
    with pytest.raises(star.StarsdError, match="INVALID_ARGUMENT"):
        h.submit(1, 0, 1, ids, q, L, tok, p=p)          # slot still in flight
    assert h.poll(timeout_us=5_000_000) == (1, 0, 0)
    assert h.poll(timeout_us=0) is None
    with pytest.raises(star.StarsdError, match="INVALID_ARGUMENT"):
        h.draft_end()                                   # end without begin
    h.close()


@pytest.mark.parametrize("N", [1, 2, 5])
def test_loopback_busy_fraction_follows_sec41_closed_form(N):
    """Draft service S and target stand-in Z as device spins (tools/star_bench.py): the measured
    draft busy fraction follows Eqs. 7-10 -- Z/S = 3 gives N_full = 4."""
    import importlib.util
    import os
    spec = importlib.util.spec_from_file_location(
        "star_bench", os.path.join(os.path.dirname(__file__), "..", "tools", "star_bench.py"))
    sb = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(sb)
    S, Z = 1.0, 3.0
    st = sb.run(N, 1, S, Z, 20, sb.sleep_cycles_per_ms(), 8, 4, 4096)
    pred = star.predicted(N, S, Z)
    assert st["rounds"] == 20 * N
    assert abs(st["busy_fraction"] - pred["busy_fraction"]) < 0.08, (st, pred)


def test_loopback_varying_batch_per_slot_and_online_predictor():
    """a slot's rounds may carry different batch sizes (B_v <= max_shape.batch);
    the slot's verify workspace must re-zero itself when the layout changes.  Rounds alternate
    B = 8, 24, 3, 24 on the same slots and every result matches the oracle.  The online predictor
    then reports S(d), Z(d) > 0 and a beta estimate from the observed accept lengths."""
    N, slots, B_max, k, V, T = 2, 2, 24, 4, 3000, 1.0
    h = star.Star(0, N + 1, B_max, k, V, T, seed=5, n_slots=slots, device=DEV, transport="loopback")
    sizes = [8, 24, 3, 24]
    inflight = {}

    def submit(v, s, r):
        B = sizes[r % len(sizes)]
        d = make_batch(V, k, B, T, 30.0, seed=500 * v + 50 * s + r)
        t = {"p": _dev(d["p"]), "q": _dev(d["q"]), "ids": _dev(d["ids"]),
             "L": torch.full((B,), -7, dtype=torch.int32, device=DEV),
             "tok": torch.full((B, k + 1), -7, dtype=torch.int32, device=DEV)}
        h.draft_begin(verifier=v)
        h.submit(v, s, r, t["ids"], t["q"], t["L"], t["tok"], request_id_base=r * 100, p=t["p"])
        h.draft_end()
        inflight[(v, s)] = (r, d, t)

    for s in range(slots):
        for v in range(1, N + 1):
            submit(v, s, 0)
    n = 0
    while inflight:
        got = h.poll(timeout_us=10_000_000)
        assert got is not None
        v, s, r = got
        r0, d, t = inflight.pop((v, s))
        L, tok = t["L"].cpu().numpy(), t["tok"].cpu().numpy()
        ref = oracle.verify(d["p"], d["q"], d["ids"], T, seed=5, round=r, rid_base=r * 100, trace=True)
        compare(d, (L, tok, np.zeros(len(L), np.int32)), ref, T, 5, r, r * 100)
        h.observe(v, L)
        n += 1
        if r + 1 < 8:
            submit(v, s, r + 1)
    assert n == N * slots * 8
    pr = h.predict(0.01)
    assert pr["service_ms"] > 0 and pr["return_ms"] > 0 and 0 < pr["expected_accepted"] < N * k
    h.close()
