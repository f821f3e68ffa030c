"""Zero-copy probe: sd_verify reading pinned (UVA-mapped) host logits directly over PCIe -- the lazy
kernels then move only the rows they need -- against the copy-everything verify_host path.
  python tools/zero_copy_probe.py [--config c3] [--steps 10]"""
import argparse
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2601_21622_b200 as sd
from paper_2601_21622_b200 import _lib
from workload import CONFIGS, make_batch_torch

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--steps", type=int, default=10)
a = ap.parse_args()
c = CONFIGS[a.config]
V, k, B, T = c["V"], c["k"], c["B"], c["T"]
dev = torch.device("cuda:0")
d = make_batch_torch(V, k, B, T, c["kappa"], c["seed"], dev)
hp = {x: (d[x].cpu().pin_memory() if d[x] is not None else None) for x in ("p", "q", "ids")}
torch.cuda.synchronize()

# reference: device-resident inputs
L0, t0, s0 = sd.verify(d["p"], d["q"] if T > 0 else None, d["ids"], T, seed=3, round=1)
torch.cuda.synchronize()

# zero copy: host pointers straight into the C ABI (pinned memory is UVA-mapped)
ws = sd.Workspace(B, k, V, T, device=dev)
L1 = torch.empty(B, dtype=torch.int32, device=dev)
t1 = torch.empty(B, k + 1, dtype=torch.int32, device=dev)
s1 = torch.empty(B, dtype=torch.int32, device=dev)
sh = _lib.Shape(B, k, V, V, V, _lib.SD_DTYPE_F32)
stream = torch.cuda.current_stream(dev)


def zc(i):
    _lib.check(_lib.load().sd_verify(hp["p"].data_ptr(), hp["q"].data_ptr() if T > 0 else None,
                                     d["ids"].data_ptr(), ctypes.byref(sh), float(T), 3, i, 0,
                                     L1.data_ptr(), t1.data_ptr(), s1.data_ptr(), ws.buf.data_ptr(),
                                     ws.nbytes, stream.cuda_stream), "sd_verify (zero copy)")


zc(1)
torch.cuda.synchronize()
same = torch.equal(L0, L1) and torch.equal(t0, t1) and torch.equal(s0, s1)
print("zero-copy outputs identical to device-resident:", same)

hout = tuple(torch.empty(x.shape, dtype=x.dtype, pin_memory=True) for x in (L1, t1, s1))
torch.cuda.synchronize()
t_start = time.perf_counter()
tok = 0
for i in range(a.steps):
    zc(i)
    for h, x in zip(hout, (L1, t1, s1)):
        h.copy_(x, non_blocking=True)
    stream.synchronize()
    tok += int((hout[0] + 1).sum())
dt = time.perf_counter() - t_start
print(f"zero copy: {dt / a.steps * 1e3:.2f} ms/step, {tok / dt:.0f} verified tokens/s")

staging = {}
sd.verify_host(hp["p"], hp["q"] if T > 0 else None, hp["ids"], T, seed=3, round=0, staging=staging)
t_start = time.perf_counter()
tok = 0
for i in range(a.steps):
    Lh, _, _ = sd.verify_host(hp["p"], hp["q"] if T > 0 else None, hp["ids"], T, seed=3, round=i,
                              staging=staging)
    tok += int((Lh + 1).sum())
dt = time.perf_counter() - t_start
print(f"verify_host (copy everything): {dt / a.steps * 1e3:.2f} ms/step, {tok / dt:.0f} verified tokens/s")
