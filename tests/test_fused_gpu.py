"""Fused sampling (k_row_stats chunk tasks sample a request's stop row one position wave after it
was read) against the tail kernel (k_sample_req) and the oracle.

The two paths share the residual arithmetic and the inverse-CDF search (cdf_search_blocks /
cdf_search_segment in csrc/verify_kernels.cu), so they must agree bit for bit on every request,
ties included; and the fused path must actually run on the Llama-3 shape (workspace word 1 counts
the requests it sampled, include/starsd.h)."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

import oracle
import paper_2601_21622_b200 as sd
from parity import compare
from workload import make_batch_torch

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda:0")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CASES = [  # (V, k, B, dtype, kappa, rgroup-independent seed)
    (128256, 7, 128, "f32", 30.0, 901),
    (128256, 7, 128, "bf16", 30.0, 902),
    (128256, 5, 96, "f32", 3.0, 903),     # low agreement: many stops at position 0
    (32000, 5, 64, "f32", 30.0, 904),
    (50000, 4, 40, "f32", 100.0, 905),    # ragged last chunk (50000 = 12 x 4096 + 848)
    (40001, 3, 24, "f32", 30.0, 906),     # ragged last vector (rows padded to 40004)
]


def _run(case, rounds):
    V, k, B, dt, kappa, seed = case
    outs = []
    fused = 0
    ws = sd.Workspace(B, k, V, 1.0, torch.float32 if dt == "f32" else torch.bfloat16, device=DEV)
    for r in range(rounds):
        if V % 4 == 0:
            b = make_batch_torch(V, k, B, 1.0, kappa, seed + r, DEV, dt)
        else:   # numpy recipe with padded rows (the torch one has no row padding)
            from workload import make_batch
            d = make_batch(V=V, k=k, B=B, T=1.0, kappa=kappa, seed=seed + r, ld=(V + 3) // 4 * 4)
            b = {x: torch.from_numpy(d[x]).to(DEV) for x in ("p", "q", "ids")}
        before = int(ws.buf[4:8].view(torch.int32).item())
        L, tok, st = sd.verify(b["p"], b["q"], b["ids"], 1.0, seed=77, round=r,
                               request_id_base=1 << 20, workspace=ws, vocab=V)
        torch.cuda.synchronize()
        fused += int(ws.buf[4:8].view(torch.int32).item()) - before
        outs.append(np.concatenate([L.cpu().numpy()[:, None], tok.cpu().numpy(),
                                    st.cpu().numpy()[:, None]], axis=1))
    return np.stack(outs), fused


_CHILD = r'''
import os, sys, json
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np
import test_fused_gpu as t
case, rounds, out = json.loads(sys.argv[1])
o, fused = t._run(tuple(case), rounds)
np.save(out, o)
print("CHILD_OK", fused)
'''


def _child(case, rounds, out, fused):
    r = subprocess.run([sys.executable, "-c", _CHILD, json.dumps([list(case), rounds, out])], cwd=ROOT,
                       env=dict(os.environ, STARSD_FUSED_SAMPLE=fused), capture_output=True,
                       text=True, timeout=900)
    assert "CHILD_OK" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]
    return np.load(out), int(r.stdout.split("CHILD_OK")[1].split()[0])


@pytest.mark.parametrize("case", CASES)
def test_fused_sampling_matches_the_tail_bit_for_bit(case, tmp_path):
    """STARSD_FUSED_SAMPLE=1 (opt-in) against the default tail sampler, one process each (the
    knob is read once per process)."""
    rounds = 6
    got, fused = _child(case, rounds, str(tmp_path / "fused.npy"), "1")
    want, none = _child(case, rounds, str(tmp_path / "tail.npy"), "0")
    V, k, B = case[0], case[1], case[2]
    assert none == 0
    if V >= 128256:
        # the Llama-3 shape: most stops are sampled inside k_row_stats
        assert fused >= rounds * B // 3, (fused, rounds * B)
    bad = np.argwhere(np.any(got != want, axis=2))
    assert bad.size == 0, (bad[:10].tolist(), got[tuple(bad[0])].tolist(), want[tuple(bad[0])].tolist())


@pytest.mark.parametrize("rgroup", ["1", "16", "48"])
def test_group_major_grid_orders_match_the_oracle(rgroup):
    """STARSD_RGROUP (group-major k_row_stats grid, a scheduling knob) changes which CTAs run the
    fused tasks, never the results: every order matches the default bit for bit and the oracle."""
    code = r'''
import os, sys, json
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np, torch
import paper_2601_21622_b200 as sd, oracle
from parity import compare
from workload import make_batch
dev = torch.device("cuda:0")
for (V, k, B, T) in [(128256, 7, 40, 1.0), (32000, 5, 64, 1.0), (128256, 7, 40, 0.0)]:
    d = make_batch(V=V, k=k, B=B, T=max(T, 1e-3), kappa=30.0, seed=V + B, ld=V)
    p, q, ids = (torch.from_numpy(d[x]).to(dev) for x in ("p", "q", "ids"))
    L, tok, st = sd.verify(p, q if T > 0 else None, ids, T, seed=5, round=9, request_id_base=3)
    torch.cuda.synchronize()
    ref = oracle.verify(d["p"], d["q"] if T > 0 else None, d["ids"], T, seed=5, round=9, rid_base=3,
                        trace=True, n_threads=8)
    s = compare(d, (L.cpu().numpy(), tok.cpu().numpy(), st.cpu().numpy()), ref, T, 5, 9, 3)
    assert s["ties"] <= max(1, 2e-2 * s["n"]), s
print("RGROUP_OK")
'''
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT,
                       env=dict(os.environ, STARSD_RGROUP=rgroup, STARSD_FUSED_SAMPLE="1"), capture_output=True, text=True,
                       timeout=900)
    assert "RGROUP_OK" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]


def test_fused_requests_match_the_oracle_at_full_size(tmp_path):
    """c3 (B = 128) with fused sampling: outputs against the oracle with the C-13 tie rule."""
    case = (128256, 7, 128, "f32", 30.0, 21622906)
    got, fused = _child(case, 1, str(tmp_path / "fused.npy"), "1")
    assert fused > 32
    b = make_batch_torch(128256, 7, 128, 1.0, 30.0, case[5], DEV, "f32")
    d = {x: b[x].cpu().numpy() for x in ("p", "q", "ids")}
    ref = oracle.verify(d["p"], d["q"], d["ids"], 1.0, seed=77, round=0, rid_base=1 << 20,
                        trace=True, n_threads=16)
    o = got[0]
    s = compare(d, (o[:, 0], o[:, 1:-1], o[:, -1]), ref, 1.0, 77, 0, 1 << 20)
    assert s["ties"] <= 1, s
