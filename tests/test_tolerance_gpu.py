"""GPU checks of north_star's numerical contract beyond token parity:

* the fp64 statistics the kernels decided with (sd_verify_trace: log-normalisers, acceptance
  ratios, residual masses) against the oracle's trace, at north_star's "probabilities and residual
  masses within 1e-5 relative" (reading C-17: |d log p| <= 1e-5, |dR| <= 1e-5 R + 5e-8);
* token parity over >= 10^4 Llama-3-shape requests with the C-13 tie budget (<= 1e-3 of requests,
  zero mismatches outside tau);
* the accept-length law Pr(L >= j) = prod_{i<j} beta_i (Lemma 1) by Monte Carlo over
  >= 10^5 Vicuna-shape requests with fresh draft samples x_j ~ q_j;
* the zero-residual fallback (C-6) forced on the device;
* a verify running beside other work on a second stream.
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
    if t is None:
        return None
    if t.dtype == torch.bfloat16:
        return t.view(torch.int16).cpu().numpy().view(np.uint16)
    return t.cpu().numpy()


def _dev(a):
    t = torch.from_numpy(np.ascontiguousarray(a))
    if a.dtype == np.uint16:
        t = t.view(torch.bfloat16)
    return t.to(DEV)


# ---------------------------------------------------------------- C-17 tolerances ----------
def _check_trace(d, T, seed=11, round=3, rid_base=500):
    p, q, ids = _dev(d["p"]), _dev(d["q"]), _dev(d["ids"])
    B, k = d["ids"].shape
    V = d["p"].shape[-1]
    ws = sd.Workspace(B, k, V, T, p.dtype, DEV)
    L, tok, st = sd.verify(p, q, ids, T, seed=seed, round=round, request_id_base=rid_base,
                           workspace=ws)
    tr_gpu = sd.verify_trace(p, L, T, ws)
    torch.cuda.synchronize()
    g = {x: v.cpu().numpy() for x, v in tr_gpu.items()}
    Lg = L.cpu().numpy()
    rL, rtok, rst, tr = oracle.verify(d["p"], d["q"], d["ids"], T, seed=seed, round=round,
                                      rid_base=rid_base, trace=True, n_threads=NTH)
    worst = dict(lam=0.0, ell=0.0, R=0.0)
    n_rows = 0
    for b in range(B):
        if rst[b] & oracle.HARD_FAULTS:
            continue
        t = tr[b]
        # rows both sides evaluated: tested positions up to min(L_gpu, L_ref)
        upto = min(int(Lg[b]), int(rL[b]))
        for j in range(min(upto + 1, k)):
            dlp = abs(g["lam_p"][b, j] - t.lam_p[j])
            dlq = abs(g["lam_q"][b, j] - t.lam_q[j])
            dell = abs(np.log(g["a"][b, j]) - t.ell[j])
            assert dlp <= 1e-5 and dlq <= 1e-5, (b, j, dlp, dlq)
            assert dell <= 2e-5, (b, j, g["a"][b, j], t.ell[j])
            worst["lam"] = max(worst["lam"], dlp, dlq)
            worst["ell"] = max(worst["ell"], dell)
            n_rows += 1
        if Lg[b] == rL[b] == k:                      # the bonus row p_k
            dl = abs(g["lam_p"][b, k] - t.lam_p[k])
            assert dl <= 1e-5, (b, "bonus", dl)
        if Lg[b] == rL[b]:                           # residual (or bonus / C-6) mass
            dR = abs(g["R"][b] - t.R)
            assert dR <= 1e-5 * t.R + 5e-8, (b, g["R"][b], t.R)
            worst["R"] = max(worst["R"], dR / max(t.R, 1e-300))
    assert n_rows > 0
    return worst


@pytest.mark.parametrize("cfg,dtype", [("c2", "f32"), ("c2", "bf16"), ("c3", "f32"), ("c3", "bf16")])
def test_statistics_within_north_star_tolerance(cfg, dtype):
    c = CONFIGS[cfg]
    B = c["B"] if cfg == "c2" else 32
    if cfg == "c2":
        d = make_batch(V=c["V"], k=c["k"], B=B, T=1.0, kappa=c["kappa"], seed=c["seed"] + 77,
                       dtype=dtype)
    else:
        t = make_batch_torch(V=c["V"], k=c["k"], B=B, T=1.0, kappa=c["kappa"],
                             seed=c["seed"] + 77, device=DEV, dtype=dtype)
        d = {x: _host(t[x]) for x in ("p", "q", "ids")}
    worst = _check_trace(d, 1.0)
    print(cfg, dtype, "worst |dlam|, |dlog a|, |dR|/R:", worst)


def test_statistics_tolerance_temperatures_and_agreement():
    """T = 0.5 / 2 and high agreement (kappa = 1000: beta ~ 0.95, p - q cancellation in R)."""
    for T, kappa in ((0.5, 30.0), (2.0, 30.0), (1.0, 1000.0)):
        d = make_batch(V=32000, k=5, B=48, T=T, kappa=kappa, seed=int(1000 * T + kappa))
        _check_trace(d, T)


# ---------------------------------------------------------------- tie budget ---------------
def test_parity_c3_ten_thousand_requests():
    """>= 10^4 Llama-3-shape requests (80 batches of B = 128, fresh rows each): every request
    bit-exact outside C-13 ties, ties <= 1e-3 of requests."""
    c = CONFIGS["c3"]
    n = ties = 0
    Ls = []
    for i in range(80):
        t = make_batch_torch(V=c["V"], k=c["k"], B=c["B"], T=1.0, kappa=c["kappa"],
                             seed=c["seed"] + 5000 + i, device=DEV)
        L, tok, st = sd.verify(t["p"], t["q"], t["ids"], 1.0, seed=21622, round=i,
                               request_id_base=i * 128)
        torch.cuda.synchronize()
        gpu = (L.cpu().numpy(), tok.cpu().numpy(), st.cpu().numpy())
        d = {x: _host(t[x]) for x in ("p", "q", "ids")}
        del t
        ref = oracle.verify(d["p"], d["q"], d["ids"], 1.0, seed=21622, round=i,
                            rid_base=i * 128, trace=True, n_threads=NTH)
        s = compare(d, gpu, ref, 1.0, 21622, i, i * 128)
        n += s["n"]
        ties += s["ties"]
        Ls.append(gpu[0])
    print("c3 requests", n, "ties", ties, "mean L", float(np.mean(np.concatenate(Ls))))
    assert n >= 10_000
    assert ties <= 1e-3 * n


def test_parity_c3_bf16_greedy():
    c = CONFIGS["c3"]
    t = make_batch_torch(V=c["V"], k=c["k"], B=c["B"], T=0.0, kappa=c["kappa"],
                         seed=c["seed"] + 31, device=DEV, dtype="bf16")
    L, tok, st = sd.verify(t["p"], None, t["ids"], 0.0)
    torch.cuda.synchronize()
    d = {x: _host(t[x]) for x in ("p", "ids")}
    d["q"] = None
    ref = oracle.verify(d["p"], None, d["ids"], 0.0, trace=True, n_threads=NTH)
    s = compare(d, (L.cpu().numpy(), tok.cpu().numpy(), st.cpu().numpy()), ref, 0.0, 0, 0, 0)
    assert s["ties"] == 0


# ---------------------------------------------------------------- accept-length law --------
def test_monte_carlo_accept_length_law():
    """Pr(L >= j) = prod_{i<j} beta_i (Lemma 1; pin P6/P7) over 1600 rounds x 64
    Vicuna-shape requests = 102400 requests: fixed rows, fresh draft samples x_j ~ q_j every round
    (torch.multinomial on the fp64 softmax), beta from the oracle (Eq. 1, fp64)."""
    from scipy import stats as st
    c = CONFIGS["c2"]
    V, k, B, T, R = c["V"], c["k"], c["B"], 1.0, 1600
    d = make_batch(V=V, k=k, B=B, T=T, kappa=c["kappa"], seed=c["seed"] + 404)
    beta = np.array([[oracle.beta(d["p"][b, j], d["q"][b, j], T) for j in range(k)]
                     for b in range(B)])
    p, q = _dev(d["p"]), _dev(d["q"])
    qprob = torch.softmax(q.double().reshape(B * k, V) / T, dim=-1)
    gen = torch.Generator(device=DEV)
    gen.manual_seed(4040)
    hist = torch.zeros(k + 1, dtype=torch.int64, device=DEV)
    per_req = torch.zeros(B, k + 1, dtype=torch.int64, device=DEV)
    for r in range(R):
        ids = torch.multinomial(qprob, 1, generator=gen).reshape(B, k).to(torch.int32)
        L, tok, stt = sd.verify(p, q, ids, T, seed=99, round=r, request_id_base=0)
        per_req.scatter_add_(1, L.long().unsqueeze(1), torch.ones(B, 1, dtype=torch.int64, device=DEV))
    cnt = per_req.cpu().numpy()                                  # [B][k+1] counts of L = j
    assert cnt.sum() == B * R
    # Pr(L = j) per request: prod_{i<j} beta_i * (1 - beta_j), Pr(L = k) = prod beta
    reach = np.concatenate([np.ones((B, 1)), np.cumprod(beta, axis=1)], axis=1)   # Pr(L >= j)
    pL = reach.copy()
    pL[:, :k] -= reach[:, 1:]
    for j in range(1, k + 1):
        obs = cnt[:, j:].sum()
        P = reach[:, j]
        exp_, var = R * P.sum(), R * (P * (1 - P)).sum()
        z = (obs - exp_) / np.sqrt(var)
        assert abs(z) < 5.0, (j, obs, exp_, z)
    expct = R * pL.sum(axis=0)
    g = 2 * np.sum(cnt.sum(axis=0) * np.log(np.maximum(cnt.sum(axis=0), 1) / expct))
    assert st.chi2.sf(g, k) > 1e-4, (cnt.sum(axis=0), expct)


# ---------------------------------------------------------------- C-6 on the device --------
def test_zero_residual_fallback_on_device():
    """A rejection whose residual vanishes in the kernel's fp32 arithmetic (C-6): q_0 equals p_0
    except at a low-probability draft token x whose q logit is larger by ~0.01, so
    a = p(x)/q(x) ~ 0.99 while S_q / S_p - 1 ~ 1e-9 rounds away in fp32 and every fp32 residual
    term max(0, p - q) is 0.  The round is chosen so that u_acc >= 0.995 (a rejection).  The GPU
    must reject (L = 0), report SD_FAULT_ZERO_RESIDUAL and sample from p_0; the oracle's fp64
    residual is ~1e-9 > 0, so the request is a C-13 tie and the token must lie in the oracle's
    CDF cell within tau."""
    V, k, T = 4096, 1, 1.0
    base = make_batch(V=V, k=k, B=24, T=T, kappa=30.0, seed=606)
    hits = 0
    for b in range(24):
        zp = base["p"][b:b + 1].copy()                      # [1, 2, V]
        row = zp[0, 0].astype(np.float64)
        pr = np.exp(row - row.max())
        pr /= pr.sum()
        x = int(np.argmin(np.abs(np.log(pr) - np.log(1e-7))))   # p(x) ~ 1e-7
        assert pr[x] < 1e-5 and x != int(np.argmax(row))
        zq = zp[:, :1].copy()
        zq[0, 0, x] = np.float32(row[x] + 0.01)
        ids = np.array([[x]], np.int32)
        rnd = next(r for r in range(100000) if oracle.uniforms(7, 0, r, 0)[0] >= 0.995)
        d = dict(p=zp, q=zq, ids=ids)
        L, tok, st = sd.verify(_dev(zp), _dev(zq), _dev(ids), T, seed=7, round=rnd,
                               request_id_base=0)
        torch.cuda.synchronize()
        gpu = (L.cpu().numpy(), tok.cpu().numpy(), st.cpu().numpy())
        assert gpu[0][0] == 0
        ref = oracle.verify(zp, zq, ids, T, seed=7, round=rnd, rid_base=0, trace=True)
        # the oracle's fp64 residual is ~1e-9: a tie (R < 5e-8), judged by the C-13 tie rule
        assert ref[0][0] == 0 and (ref[3][0].R < 5e-8 or ref[2][0] & 16)
        compare(d, gpu, ref, T, 7, rnd, 0)
        hits += int(gpu[2][0] & sd.FAULT_ZERO_RESIDUAL != 0)
    assert hits >= 20, hits


# ---------------------------------------------------------------- concurrency --------------
def test_verify_beside_other_work_on_a_second_stream():
    """sd_verify on one stream while other kernels run on a second stream (and a second verify
    with its own workspace): no dispatch-order assumption may break (tagged rows' deciders wait
    only on CTAs that started before them), results equal the oracle's."""
    c = CONFIGS["c3"]
    t = make_batch_torch(V=c["V"], k=c["k"], B=24, T=1.0, kappa=c["kappa"], seed=c["seed"] + 99,
                         device=DEV)
    t2 = make_batch_torch(V=32000, k=5, B=64, T=1.0, kappa=30.0, seed=1717, device=DEV)
    s1, s2 = torch.cuda.Stream(DEV), torch.cuda.Stream(DEV)
    a = torch.randn(8192, 8192, device=DEV, dtype=torch.bfloat16)
    torch.cuda.synchronize()
    outs = []
    for it in range(4):
        with torch.cuda.stream(s2):
            for _ in range(3):
                a = (a @ a).clamp_(-1, 1)
            L2, tok2, st2 = sd.verify(t2["p"], t2["q"], t2["ids"], 1.0, seed=5, round=it,
                                      stream=s2)
        with torch.cuda.stream(s1):
            L, tok, st = sd.verify(t["p"], t["q"], t["ids"], 1.0, seed=5, round=it, stream=s1)
        outs.append(((L, tok, st), (L2, tok2, st2), it))
    torch.cuda.synchronize()
    d = {x: _host(t[x]) for x in ("p", "q", "ids")}
    d2 = {x: _host(t2[x]) for x in ("p", "q", "ids")}
    for (g1, g2, it) in outs:
        for dd, g in ((d, g1), (d2, g2)):
            ref = oracle.verify(dd["p"], dd["q"], dd["ids"], 1.0, seed=5, round=it, trace=True,
                                n_threads=NTH)
            compare(dd, tuple(x.cpu().numpy() for x in g), ref, 1.0, 5, it, 0)
