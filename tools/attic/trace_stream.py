"""Event timeline of one stream-kernel sd_verify call (sd_debug_trace) -> gpurun_out/strace_<cfg>.npz.
Usage on the box: python tools/trace_stream.py --config c3"""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2601_21622_b200 as sd
from paper_2601_21622_b200 import _lib
from workload import CONFIGS, make_batch_torch

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--dtype", default="f32")
ap.add_argument("--out", default="gpurun_out")
a = ap.parse_args()
c = CONFIGS[a.config]
T = c["T"]
dev = torch.device("cuda:0")
bs = [make_batch_torch(c["V"], c["k"], c["B"], T, c["kappa"], c["seed"] + i, dev, a.dtype) for i in range(4)]
pl = sd.plan(c["B"], c["k"], c["V"], T, torch.float32 if a.dtype == "f32" else torch.bfloat16)
grid = pl["ctas"]
N = 8192
buf = torch.zeros(grid * N, dtype=torch.int64, device=dev)
for i in range(6):
    b = bs[i % 4]
    sd.verify(b["p"], b["q"] if T > 0 else None, b["ids"], T, seed=1, round=i)
torch.cuda.synchronize()
_lib.load().sd_debug_trace(buf.data_ptr())
b = bs[1]
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
L, tok, st = sd.verify(b["p"], b["q"] if T > 0 else None, b["ids"], T, seed=1, round=99)
e1.record()
torch.cuda.synchronize()
_lib.load().sd_debug_trace(None)
print("plan", pl, "call us", e0.elapsed_time(e1) * 1e3, "mean L", float(L.float().mean()))
np.savez(os.path.join(a.out, f"strace_{a.config}_{a.dtype}.npz"), buf=buf.cpu().numpy().reshape(grid, N),
         L=L.cpu().numpy(), C=pl["cluster"], B=c["B"], k=c["k"])
