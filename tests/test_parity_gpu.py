"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on identical seeded
inputs, element by element (rule C-13 in tests/parity.py)."""
import os

import numpy as np
import pytest
import torch

import oracle
from parity import compare
from workload import CONFIGS, make_batch, make_batch_torch, make_tiny_tables, tiny_batch

pytestmark = pytest.mark.gpu

sd = pytest.importorskip("paper_2601_21622_b200")
DEV = torch.device("cuda:0")
NTH = max(1, min(8, len(os.sched_getaffinity(0))))


def run_both(d, T, seed=1234, round=5, rid_base=1000, V=None, dtype=torch.float32):
    """Run the GPU path and the oracle on the same numpy inputs."""
    def dev(a):
        if a is None:
            return None
        t = torch.from_numpy(np.ascontiguousarray(a))
        if a.dtype == np.uint16:
            t = t.view(torch.bfloat16)
        return t.to(DEV)
    p, q, ids = dev(d["p"]), dev(d["q"]) if T > 0 else None, dev(d["ids"])
    L, tok, st = sd.verify(p, q, ids, T, seed=seed, round=round, request_id_base=rid_base,
                           vocab=V)
    torch.cuda.synchronize()
    gpu = (L.cpu().numpy(), tok.cpu().numpy(), st.cpu().numpy())
    ref = oracle.verify(d["p"], d["q"] if T > 0 else None, d["ids"], T, seed=seed, round=round,
                        rid_base=rid_base, V=V, trace=True, n_threads=NTH)
    return gpu, ref


def check(d, T, max_tie_frac=1e-3, **kw):
    gpu, ref = run_both(d, T, **kw)
    stats = compare(d, gpu, ref, T, kw.get("seed", 1234), kw.get("round", 5),
                    kw.get("rid_base", 1000), V=kw.get("V"))
    assert stats["ties"] <= max(1, max_tie_frac * stats["n"]), stats
    return gpu, ref, stats


# ---------------------------------------------------------------- Philox on the device -----
def test_device_philox_known_answers_and_stream():
    kat = [l.split() for l in open(os.path.join(os.path.dirname(__file__), "golden",
                                                "philox4x32_10_kat.txt"))
           if l.strip() and not l.startswith("#")]
    for r in kat:
        v = [int(x, 16) for x in r]
        seed = v[4] | (v[5] << 32)
        rid = v[2] | (v[3] << 32)
        w = sd.philox_words(seed, v[1], torch.tensor([v[0]], dtype=torch.int64).to(torch.int32).to(DEV),
                            torch.tensor([rid - (1 << 64) if rid >= (1 << 63) else rid],
                                         dtype=torch.int64, device=DEV))
        assert w[0].tolist() == v[6:10]
    rng = np.random.default_rng(0)
    n = 4096
    pos = rng.integers(0, 32, n)
    rid = rng.integers(0, 2**62, n)
    w = sd.philox_words(99, 17, torch.from_numpy(pos.astype(np.int32)).to(DEV),
                        torch.from_numpy(rid.astype(np.int64)).to(DEV)).cpu().numpy()
    for i in range(0, n, 7):
        ref = oracle.philox([pos[i], 17, rid[i] & 0xFFFFFFFF, rid[i] >> 32], [99, 0])
        assert list(w[i]) == list(ref)


# ---------------------------------------------------------------- configs -----------------
def test_parity_c1_tiny_exhaustive_paths():
    """C1: V=8, k=4, all 8^4 draft paths through prefix-conditioned tables, several rounds."""
    P, Q = make_tiny_tables(V=8, k=4, seed=21622001)
    paths = np.array(np.meshgrid(*[np.arange(8)] * 4, indexing="ij")).reshape(4, -1).T
    p, q = tiny_batch(P, Q, paths.astype(np.int32))
    d = dict(p=p, q=q, ids=paths.astype(np.int32))
    for rnd in range(3):
        check(d, 1.0, round=rnd, max_tie_frac=1e-2)
    check(d, 0.7, round=9, max_tie_frac=1e-2)
    check(d, 0.0)


@pytest.mark.parametrize("T", [1.0, 0.0])
def test_parity_c2_vicuna_full(T):
    c = CONFIGS["c2"]
    d = make_batch(V=c["V"], k=c["k"], B=c["B"], T=T, kappa=c["kappa"], seed=c["seed"])
    gpu, ref, stats = check(d, T)
    assert 0 < np.mean(ref[0]) < c["k"]


@pytest.mark.parametrize("kappa", [3.0, 300.0])
def test_parity_c2_agreement_sweep(kappa):
    d = make_batch(V=32000, k=5, B=64, T=1.0, kappa=kappa, seed=21622002 + int(kappa))
    check(d, 1.0)


def test_parity_c2_bf16():
    d = make_batch(V=32000, k=5, B=64, T=1.0, kappa=30.0, seed=21622012, dtype="bf16")
    check(d, 1.0)
    d = make_batch(V=32000, k=5, B=64, T=0.0, kappa=30.0, seed=21622013, dtype="bf16")
    check(d, 0.0)


def _torch_batch(cfg, T, B=None, dtype="f32", seed_off=0):
    c = CONFIGS[cfg]
    d = make_batch_torch(V=c["V"], k=c["k"], B=B or c["B"], T=T, kappa=c["kappa"],
                         seed=c["seed"] + seed_off, device=DEV, dtype=dtype)
    def host(t):
        if t.dtype == torch.bfloat16:
            return t.view(torch.int16).cpu().numpy().view(np.uint16)
        return t.cpu().numpy()
    return dict(p=host(d["p"]), q=host(d["q"]), ids=d["ids"].cpu().numpy())


@pytest.mark.parametrize("T", [1.0, 0.0])
def test_parity_c3_llama3_full(T):
    """C3 at its full size (V=128256, k=7, B=128): every request compared."""
    d = _torch_batch("c3", T)
    gpu, ref, stats = check(d, T)
    print("c3", T, stats, "mean L", np.mean(ref[0]))


def test_parity_c3_bf16():
    d = _torch_batch("c3", 1.0, B=32, dtype="bf16", seed_off=7)
    check(d, 1.0)


# ---------------------------------------------------------------- edge cases --------------
@pytest.mark.parametrize("V,k,B", [(2, 1, 64), (8, 31, 16), (1003, 3, 50), (4097, 2, 33),
                                   (12345, 6, 9), (32768, 1, 5),
                                   # more requests than SMs: the early sampler's CTAs (and its
                                   # completion probe) run in several waves behind k_row_stats
                                   (4096, 2, 400), (40000, 3, 1), (70000, 1, 160)])
def test_parity_ragged_shapes(V, k, B):
    """Vocabularies that are not multiples of the vector/tile/chunk sizes, k at its extremes."""
    ld = (V + 3) // 4 * 4          # rows 16-byte aligned
    d = make_batch(V=V, k=k, B=B, T=1.0, kappa=10.0, seed=V + k, ld=ld)
    check(d, 1.0, V=V, max_tie_frac=2e-2)
    check(d, 0.0, V=V)
    check(d, 0.5, V=V, max_tie_frac=2e-2)


def test_padding_is_never_read():
    """ld > V with NaN padding: a kernel reading past V would report NONFINITE."""
    d = make_batch(V=5000, k=4, B=32, T=1.0, kappa=30.0, seed=77, ld=5120)
    gpu, ref, _ = check(d, 1.0, V=5000)
    assert np.all(gpu[2] == 0)


def test_empty_batch_is_a_no_op():
    p = torch.zeros(0, 3, 64, device=DEV)
    q = torch.zeros(0, 2, 64, device=DEV)
    ids = torch.zeros(0, 2, dtype=torch.int32, device=DEV)
    L, tok, st = sd.verify(p, q, ids, 1.0)
    assert L.numel() == 0


def test_faults_follow_the_oracle():
    d = make_batch(V=3000, k=4, B=8, T=1.0, kappa=30.0, seed=13)
    p, q, ids = d["p"].copy(), d["q"].copy(), d["ids"].copy()
    p[0, 0, 5] = np.nan                      # NONFINITE at position 0
    ids[1, 0] = 3000                         # bad draft id
    p[2, 0, ids[2, 0]] = -np.inf             # certain rejection at 0 ...
    p[2, 2, 7] = np.nan                      # ... so this NaN is never reached (laziness)
    q[3, 0, :] = -np.inf                     # empty q row
    q[4, 0, ids[4, 0]] = -np.inf             # q(x) = 0 -> ZERO_Q rejection
    p[5, 1, 9] = np.inf                      # +inf at position 1 (reached if 0 accepted)
    ids[6, 3] = -5                           # bad id at a later position
    p[7, 4, :] = -np.inf                     # empty bonus row (reached only on full accept)
    dd = dict(p=p, q=q, ids=ids)
    gpu, ref, _ = check(dd, 1.0)
    assert gpu[2][0] == oracle.FAULT_NONFINITE and gpu[2][1] == oracle.FAULT_BAD_DRAFT_ID
    assert gpu[2][3] == oracle.FAULT_EMPTY_ROW and gpu[2][4] == oracle.FAULT_ZERO_Q
    assert gpu[2][2] == 0 and gpu[0][2] == 0
    pg = p.copy()
    pg[0, 0, 5] = np.nan
    check(dict(p=pg, q=None, ids=ids), 0.0)


def test_identical_rows_and_disjoint_one_hots():
    d = make_batch(V=20000, k=5, B=40, T=1.0, kappa=30.0, seed=21)
    q = d["p"][:, :5].copy()
    ids = np.argmax(q, -1).astype(np.int32)
    gpu, ref, _ = check(dict(p=d["p"], q=q, ids=ids), 1.0)
    assert np.all(gpu[0] == 5)
    V, k = 4096, 3
    p = np.full((16, k + 1, V), -np.inf, np.float32)
    qq = np.full((16, k, V), -np.inf, np.float32)
    p[:, :, 4000] = 0.0
    qq[:, :, 17] = 0.0
    ids = np.full((16, k), 17, np.int32)
    gpu, ref, _ = check(dict(p=p, q=qq, ids=ids), 1.0)
    assert np.all(gpu[0] == 0) and np.all(gpu[1][:, 0] == 4000)


def test_workspace_left_zeroed_and_deterministic():
    d = make_batch(V=32000, k=5, B=64, T=1.0, kappa=30.0, seed=5)
    p, q, ids = (torch.from_numpy(d[x]).to(DEV) for x in ("p", "q", "ids"))
    ws = sd.Workspace(64, 5, 32000, 1.0, device=DEV)
    outs = []
    for _ in range(3):
        outs.append([t.cpu() for t in sd.verify(p, q, ids, 1.0, seed=3, workspace=ws)])
    torch.cuda.synchronize()
    for o in outs[1:]:
        for a, b in zip(o, outs[0]):
            assert torch.equal(a, b)
    assert int(ws.buf[16:64 * 4 * 8].abs().sum()) == 0  # rej masks and tickets are zero again
    # (bytes 0..15: the call counter tagged partials derive their tags from)


def test_gpu_monte_carlo_matches_exact_outcome():
    """Distributional check of the GPU path itself: one tiny request replicated over 2^17
    request ids; G-test of the (L, token) histogram against the oracle's exact distribution."""
    from scipy import stats as st
    rng = np.random.default_rng(3)
    V, k, B = 8, 4, 1 << 17
    zp = rng.normal(0, 1.2, (1, k + 1, V)).astype(np.float32)
    zq = rng.normal(0, 1.2, (1, k, V)).astype(np.float32)
    ids = np.array([[2, 5, 1, 7]], np.int32)
    exact = oracle.outcome_dist(zp, zq, ids, 1.0)[0].ravel()
    p = torch.from_numpy(zp).to(DEV).expand(B, -1, -1).contiguous()
    q = torch.from_numpy(zq).to(DEV).expand(B, -1, -1).contiguous()
    L, tok, _ = sd.verify(p, q, torch.from_numpy(ids).to(DEV).expand(B, -1).contiguous(), 1.0,
                          seed=11)
    L = L.cpu().numpy()
    t = tok.cpu().numpy()[np.arange(B), L]
    obs = np.bincount(L * V + t, minlength=(k + 1) * V)
    keep = exact * B > 5
    g = 2 * np.sum(obs[keep] * np.log(np.maximum(obs[keep], 1) / (B * exact[keep])))
    assert st.chi2.sf(g, keep.sum() - 1) > 1e-4


@pytest.mark.parametrize("env,want", [
    ({"STARSD_ROWCLUSTER": "1"}, ("two_launch", 0)),        # cluster-free k_row_stats
    ({"STARSD_ROWCLUSTER": "-8"}, ("two_launch", 8)),       # clusters of 8 on every row (G > 1)
    ({"STARSD_ROWCLUSTER": "-2"}, ("two_launch", 2)),
    ({"STARSD_PUBLISH_TICKET": "1"}, ("two_launch", 0)),   # release-ordered partials + row ticket
    ({"STARSD_RGROUP": "5"}, ("two_launch", 0)),           # group-major k_row_stats grid
    ({"STARSD_EARLY": "0"}, ("two_launch", 0)),            # sampler after k_row_stats completes
])
def test_kernel_variants_match_the_oracle(env, want):
    """Kernel variants chosen by environment (once per process, so in a subprocess) against the
    oracle on the default path's cases plus a Llama-3-vocabulary case: the tail sampler after
    k_row_stats completes (no early launch), the cluster-free k_row_stats (tagged partials), forced
    clusters whose row partials meet through the global ticket (G = ceil(nch / CL) > 1), and the
    ticket publish."""
    import json
    import subprocess
    import sys
    code = r'''
import os, sys, json
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np, torch
import paper_2601_21622_b200 as sd
import oracle
from parity import compare
from workload import make_batch
want = json.loads(sys.argv[1])
pl = sd.plan(128, 7, 128256, 1.0)
assert pl["variant"] == want[0], pl
if want[1] is not None:
    assert pl["cluster"] == want[1], pl
for (V, k, B, T, ld, dt) in [(32000, 5, 64, 1.0, 32000, "f32"), (32000, 5, 64, 0.0, 32000, "f32"),
                             (1003, 3, 50, 1.0, 1004, "f32"), (12345, 6, 9, 0.5, 12348, "f32"),
                             (128256, 3, 6, 1.0, 128256, "f32"), (128256, 3, 6, 0.0, 128256, "f32"),
                             (128256, 4, 5, 1.0, 128256, "bf16"), (100000, 2, 7, 1.0, 100000, "bf16")]:
    d = make_batch(V=V, k=k, B=B, T=max(T, 1e-3), kappa=10.0, seed=V + k, ld=ld, dtype=dt)
    dev = torch.device("cuda:0")
    tdev = lambda a: (torch.from_numpy(a).view(torch.bfloat16) if a.dtype == np.uint16 else torch.from_numpy(a)).to(dev)
    p = tdev(d["p"]); q = tdev(d["q"]); ids = torch.from_numpy(d["ids"]).to(dev)
    L, tok, st = sd.verify(p, q if T > 0 else None, ids, T, seed=1234, round=5, request_id_base=1000, vocab=V)
    torch.cuda.synchronize()
    gpu = (L.cpu().numpy(), tok.cpu().numpy(), st.cpu().numpy())
    ref = oracle.verify(d["p"], d["q"] if T > 0 else None, d["ids"], T, seed=1234, round=5, rid_base=1000,
                        V=V, trace=True, n_threads=8)
    stats = compare(d, gpu, ref, T, 1234, 5, 1000, V=V)
    assert stats["ties"] <= max(1, 2e-2 * stats["n"]), stats
print("VARIANT_OK")
'''
    r = subprocess.run([sys.executable, "-c", code, json.dumps(list(want))],
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                       env=dict(os.environ, **env), capture_output=True, text=True, timeout=900)
    assert "VARIANT_OK" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]


@pytest.mark.parametrize("T", [1.0, 0.0])
def test_parity_vocab_beyond_the_on_chip_sampler(T):
    """V = 300000 (fp32) exceeds the per-request sampler's on-chip segment table (2048 segments
    of 128 logits): the chunked sampling kernel serves it; both must match the oracle."""
    V = 300000
    d = make_batch(V=V, k=2, B=6, T=max(T, 1e-3), kappa=10.0, seed=300000, ld=V)
    check(d, T, V=V, max_tie_frac=2e-1)


@pytest.mark.parametrize("T", [1.0, 0.0])
def test_parity_max_chain_length(T):
    """k = 31 (the ballot/mask limit): 32 positions per request at the Vicuna vocabulary."""
    d = make_batch(V=32000, k=31, B=8, T=max(T, 1e-3), kappa=300.0, seed=3131)
    check(d, T)


def test_parity_single_request_llama3_vocab():
    """B = 1 at V = 128256: one request's rows spread over the whole grid / one sampler CTA."""
    d = make_batch(V=128256, k=7, B=1, T=1.0, kappa=30.0, seed=128)
    check(d, 1.0)
    check(d, 0.0)


def test_parity_bf16_ragged_vocab_and_padding():
    """bf16 with a vocabulary that is not a multiple of the 8-logit vector, NaN-padded rows."""
    V = 12345
    d = make_batch(V=V, k=4, B=24, T=1.0, kappa=30.0, seed=12345, dtype="bf16", ld=12352)
    gpu, ref, _ = check(d, 1.0, V=V, max_tie_frac=2e-2)
    assert np.all(gpu[2] == 0)
    check(d, 0.0, V=V)


@pytest.mark.parametrize("T", [0.05, 5.0])
def test_parity_extreme_temperatures(T):
    """Very peaked (T = 0.05: c2 = log2(e)/T ~ 29) and very flat (T = 5) distributions."""
    d = make_batch(V=32000, k=5, B=32, T=T, kappa=30.0, seed=int(T * 1000) + 7)
    check(d, T, max_tie_frac=2e-2)


def test_profile_timestamps_bracket_the_stats_kernel():
    """sd_profile_timestamps (bench.py's roofline clock): for each profiled call, the earliest
    k_row_stats CTA start precedes the moment the second kernel saw it complete, by a plausible
    span; unprofiled calls leave the buffer untouched."""
    import ctypes
    from paper_2601_21622_b200 import _lib
    d = make_batch(V=32000, k=5, B=16, T=1.0, kappa=30.0, seed=77)
    dev = torch.device("cuda:0")
    p, q, ids = (torch.from_numpy(d[x]).to(dev) for x in ("p", "q", "ids"))
    ts = torch.full((3, 2), -1, dtype=torch.int64, device=dev)
    L = _lib.load()
    _lib.check(L.sd_profile_timestamps(ctypes.c_void_p(ts.data_ptr()), 2), "sd_profile_timestamps")
    try:
        sd.verify(p, q, ids, 1.0, seed=1, round=0)      # profiled: slot 0
        sd.verify(p, None, ids, 0.0, seed=1, round=0)   # profiled: slot 1 (greedy finalizer)
        sd.verify(p, q, ids, 1.0, seed=1, round=1)      # past n_calls: not profiled
    finally:
        _lib.check(L.sd_profile_timestamps(None, 0), "sd_profile_timestamps")
    torch.cuda.synchronize()
    t = ts.cpu().numpy().view(np.uint64)
    for i in range(2):                               # the sampled call and the greedy call
        assert t[i, 0] != np.uint64(2**64 - 1) and t[i, 1] != np.uint64(2**64 - 1)
        span = int(t[i, 1]) - int(t[i, 0])
        assert 0 < span < 10_000_000, span           # ns
    assert (t[2] == np.uint64(2**64 - 1)).all()      # only n_calls calls are profiled
    with pytest.raises(sd.StarsdError):
        _lib.check(L.sd_profile_timestamps(None, 3), "sd_profile_timestamps")


def test_one_workspace_serves_shapes_of_different_layout():
    """A workspace sized for a large shape serves any sequence of smaller shapes of a different
    layout (tagged partials, clusters, tickets) with no caller action: the library re-zeroes the
    union of the two zero regions when the shape changes (include/starsd.h: the star's
    per-slot workspaces see varying batch sizes)."""
    ws = sd.Workspace(16, 7, 128256, 1.0, device=DEV)
    cases = [(128256, 7, 16, 1.0), (128256, 7, 16, 1.0), (60000, 3, 8, 1.0), (32000, 5, 12, 1.0),
             (128256, 7, 16, 0.0), (300000, 2, 2, 1.0), (128256, 7, 16, 1.0), (128256, 7, 4, 1.0),
             (128256, 7, 16, 1.0), (32000, 5, 3, 0.0), (32000, 5, 12, 1.0)]
    for i, (V, k, B, T) in enumerate(cases):
        d = make_batch(V=V, k=k, B=B, T=max(T, 1e-3), kappa=30.0, seed=900 + i)
        p, q, ids = (torch.from_numpy(d[x]).to(DEV) for x in ("p", "q", "ids"))
        assert sd.workspace_size(B, k, V, T) <= ws.nbytes
        L, tok, st = sd.verify(p, q if T > 0 else None, ids, T, seed=4, round=i, workspace=ws)
        torch.cuda.synchronize()
        ref = oracle.verify(d["p"], d["q"] if T > 0 else None, d["ids"], T, seed=4, round=i,
                            trace=True, n_threads=8)
        stats = compare(d, (L.cpu().numpy(), tok.cpu().numpy(), st.cpu().numpy()), ref, T, 4, i, 0)
        assert stats["ties"] <= max(1, 2e-2 * stats["n"]), stats


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_verify_host_zero_copy_and_copy_paths_match_the_device_call(dtype):
    """verify_host: pinned host logits are read in place by the kernels (zero copy), unpinned ones
    are copied first; both must equal the device-resident call bit for bit, sampled and greedy,
    and one staging dict must survive switching between them (and between T = 0 and T > 0)."""
    d = make_batch_torch(V=128256, k=7, B=24, T=1.0, kappa=30.0, seed=77, device=DEV, dtype=dtype)
    staging = {}
    for T in (1.0, 0.0, 1.0):
        q = d["q"] if T > 0 else None
        ref = [t.cpu() for t in sd.verify(d["p"], q, d["ids"], T, seed=5, round=2, request_id_base=9)]
        torch.cuda.synchronize()
        for pinned in (True, False):
            hp = d["p"].cpu().pin_memory() if pinned else d["p"].cpu()
            hq = None if q is None else (q.cpu().pin_memory() if pinned else q.cpu())
            got = sd.verify_host(hp, hq, d["ids"].cpu(), T, seed=5, round=2, request_id_base=9,
                                 staging=staging)
            assert (staging["p"] is None) == pinned                      # the path taken
            for a, b in zip(got, ref):
                assert torch.equal(a, b), (dtype, T, pinned)
