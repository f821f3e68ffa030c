"""Small verify / draft calls for compute-sanitizer (memcheck, racecheck, synccheck):
  compute-sanitizer --tool memcheck python tools/sanitize_run.py
Every kernel of the library runs at least once on shapes that take each publish path (single-chunk
ticket rows, whole-row clusters, tagged rows), the chunked and on-chip samplers, greedy, the draft
sampler and the lazy-q verify."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2601_21622_b200 as sd
from workload import make_batch

dev = torch.device("cuda:0")
for (V, k, B, T) in ((8, 4, 3, 1.0), (3000, 3, 4, 1.0), (32000, 5, 4, 1.0), (32000, 5, 4, 0.0),
                     (128256, 7, 2, 1.0), (128256, 7, 2, 0.0), (300000, 2, 2, 1.0)):
    d = make_batch(V=V, k=k, B=B, T=max(T, 1e-3), kappa=30.0, seed=V + k)
    p, q, ids = (torch.from_numpy(d[x]).to(dev) for x in ("p", "q", "ids"))
    L, tok, st = sd.verify(p, q if T > 0 else None, ids, T, seed=1, round=2)
    if T > 0:
        ids2, qm, _ = sd.draft_sample(q, T, seed=1, round=2)
        sd.verify_qmeta(p, q, qm, ids2, T, seed=1, round=2)
    torch.cuda.synchronize()
    print("ok", V, k, B, T, L.tolist(), flush=True)
print("SANITIZE_RUN_DONE")
