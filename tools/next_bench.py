"""Measurement of the NEXT rows on one B200, one JSON line each:
  NEXT-2  sd_draft_sample: draft tokens drawn per second from the q rows of a c3 batch;
  NEXT-1  sd_verify_qmeta (lazy q) against sd_verify on the same c3 batch;
  NEXT-3  sd_tree_verify: full binary trees of depth 4 at V = 128256.
Time: CUDA events around `--iters` back-to-back calls (after warm-up) on two rotated input sets
(> L2).  Bytes: the rows each call must read once (algorithmic, SURVEY 8(d) style), divided by
the time, against MEASURED_PEAKS.json's copy bandwidth.
  python tools/next_bench.py [--iters 50]"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

import paper_2601_21622_b200 as sd
from workload import CONFIGS, make_batch_torch

ap = argparse.ArgumentParser()
ap.add_argument("--iters", type=int, default=50)
a = ap.parse_args()
dev = torch.device("cuda:0")
try:
    PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
except Exception:
    PEAK = 6650.0


def timed(fn, n):
    for i in range(3):
        fn(i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(n):
        fn(i)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


def line(name, ms, units, unit, alg_bytes, extra):
    gbs = alg_bytes / (ms / 1000.0) / 1e9
    print(json.dumps({"row": name, "ms_per_call": ms, "value": units / (ms / 1000.0), "unit": unit,
                      "alg_bytes_per_call": alg_bytes, "achieved_gbs": gbs, "peak_gbs": PEAK,
                      "frac": gbs / PEAK, **extra}), flush=True)


c = CONFIGS["c3"]
V, k, B = c["V"], c["k"], c["B"]
bs = [make_batch_torch(V, k, B, 1.0, c["kappa"], c["seed"] + i, dev) for i in range(2)]
torch.cuda.synchronize()

# NEXT-2: draw x_j ~ softmax(q_j) for all B*k rows (statistics pass + inverse-CDF pass per row)
ms = timed(lambda i: sd.draft_sample(bs[i % 2]["q"], 1.0, seed=1, round=i), a.iters)
line("NEXT-2 sd_draft_sample (c3 q rows)", ms, B * k, "draft tokens/s", 2.0 * B * k * V * 4,
     {"shape": {"B": B, "k": k, "V": V}, "bytes_note": "each q row read twice (statistics, sample)"})

# NEXT-1: lazy q -- the verifier reads q only at the stop row
qms = []
for b in bs:
    ids, qm, _ = sd.draft_sample(b["q"], 1.0, seed=2, round=0)
    b["ids2"], b["qm"] = ids, qm
    qms.append(qm)
torch.cuda.synchronize()
Ls = []


def full(i):
    b = bs[i % 2]
    Ls.append(sd.verify(b["p"], b["q"], b["ids2"], 1.0, seed=3, round=i)[0])


def lazy(i):
    b = bs[i % 2]
    Ls.append(sd.verify_qmeta(b["p"], b["q"], b["qm"], b["ids2"], 1.0, seed=3, round=i)[0])


ms_full = timed(full, a.iters)
Lf = torch.stack(Ls[-a.iters:]).cpu().numpy()
Ls.clear()
ms_lazy = timed(lazy, a.iters)
Lz = torch.stack(Ls[-a.iters:]).cpu().numpy()
alg_full = float(((Lf + 1) * V * 4 + np.minimum(Lf + 1, k) * V * 4).sum(axis=1).mean())
alg_lazy = float(((Lz + 1) * V * 4 + (Lz < k) * V * 4).sum(axis=1).mean())   # p rows + one q row
line("NEXT-1 sd_verify_qmeta (lazy q, c3)", ms_lazy, float((Lz + 1).sum(axis=1).mean()),
     "verified tokens/s", alg_lazy, {"vs_full_q_ms": ms_full, "full_q_alg_bytes": alg_full,
                                     "bytes_note": "p rows 0..L + the stop q row"})

# NEXT-3: full binary trees of depth 4 (31 nodes) at the Llama-3 vocabulary
m, d, Bt = 2, 4, 32
N, Nint = 2 ** (d + 1) - 1, 2 ** d - 1
trees = []
for i in range(2):
    t = make_batch_torch(V, N - 1, Bt, 1.0, c["kappa"], 777 + i, dev)
    p, q = t["p"], t["q"][:, :Nint].contiguous()
    g = torch.Generator(device=dev)
    g.manual_seed(99 + i)
    tok = torch.zeros(Bt, N, dtype=torch.int32, device=dev)
    for n in range(Nint):
        for j in range(m):   # each child's token: a Gumbel-max draw from the parent's draft row
            u = torch.rand(Bt, V, generator=g, device=dev, dtype=torch.float64).clamp_min(1e-300)
            tok[:, m * n + 1 + j] = torch.argmax(q[:, n].double() - torch.log(-torch.log(u)), dim=-1).int()
    trees.append((p, q, tok))
torch.cuda.synchronize()
Lt = []
ms = timed(lambda i: Lt.append(sd.tree_verify(*trees[i % 2], m, 1.0, seed=4, round=i)[0]), a.iters)
Lt = torch.stack(Lt[-a.iters:]).cpu().numpy()
alg = float(((Lt + 1) * V * 4 + np.minimum(Lt + 1, d) * V * 4).sum(axis=1).mean())
line("NEXT-3 sd_tree_verify (m 2, depth 4, V 128256, B 32)", ms, float((Lt + 1).sum(axis=1).mean()),
     "verified tokens/s", alg, {"mean_depth": float(Lt.mean()),
                                "bytes_note": "p rows of the visited nodes + q rows of the visited internal nodes"})
