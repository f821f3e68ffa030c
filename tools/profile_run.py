"""Eager sd_verify loop for ncu: `ncu ... python tools/profile_run.py --config c2 --calls 30`.
Rotates 8 resident batches like bench.py (no CUDA graph, so every launch is a plain kernel)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2601_21622_b200 as sd
from workload import CONFIGS, make_batch_torch

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--calls", type=int, default=30)
ap.add_argument("--dtype", default="f32")
ap.add_argument("--temperature", type=float, default=None)
ap.add_argument("--nbatch", type=int, default=8)
a = ap.parse_args()
c = CONFIGS[a.config]
T = c["T"] if a.temperature is None else a.temperature
dev = torch.device("cuda:0")
bs = [make_batch_torch(c["V"], c["k"], c["B"], T, c["kappa"], c["seed"] + i, dev, a.dtype)
      for i in range(a.nbatch)]
torch.cuda.synchronize()
for i in range(a.calls):
    b = bs[i % a.nbatch]
    L, tok, st = sd.verify(b["p"], b["q"] if T > 0 else None, b["ids"], T, seed=1, round=i)
torch.cuda.synchronize()
print("mean L", float(L.float().mean()))
