"""Small reproducer of one sd_verify call on GPU (debugging aid): python tools/repro_small.py V k B T"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2601_21622_b200 as sd
from workload import make_batch

V, k, B, T = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), float(sys.argv[4])
ld = (V + 3) // 4 * 4
d = make_batch(V=V, k=k, B=B, T=max(T, 1e-3), kappa=10.0, seed=7, ld=ld)
dev = torch.device("cuda:0")
p = torch.from_numpy(d["p"]).to(dev)
q = torch.from_numpy(d["q"]).to(dev)
ids = torch.from_numpy(d["ids"]).to(dev)
print("plan", sd.plan(B, k, V, T), flush=True)
L, tok, st = sd.verify(p, q if T > 0 else None, ids, T, seed=1, round=0, vocab=V)
torch.cuda.synchronize()
print("ok mean L", float(L.float().mean()), "status", int(st.abs().sum()), flush=True)
