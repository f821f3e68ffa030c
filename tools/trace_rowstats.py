"""Per-CTA phase timeline of one two-launch sd_verify call (debug build: STARSD_BUILD_DEBUG=1,
sd_debug_trace) -> gpurun_out/rtrace_<cfg>_<dtype>.npz, plus a printed summary.

k_row_stats record (8 words per CTA, %globaltimer ns): 0 start, 1 after stop-mask read,
2 p slice arrived, 3 q slice arrived, 4 block reduction done, 5 published (ticket taken),
6 end, 7 = smid << 32 | flags (1 skipped, 2 last arriver).  k_sample_req: 0 start, 1 after
griddepcontrol.wait, 2 end, 3 first unit staged, 4 row streamed, 5 block/segment search done.
Usage on the box: python tools/trace_rowstats.py --config c3
"""
import argparse
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2601_21622_b200 as sd  # noqa: E402
from paper_2601_21622_b200 import _lib  # noqa: E402
from workload import CONFIGS, make_batch_torch  # noqa: E402


def summarize(d):
    tr, nA, B, k, nch = d["tr"], int(d["nA"]), int(d["B"]), int(d["k"]), int(d["nch"])
    A = tr[:nA].astype(np.int64)
    S = tr[nA:nA + B].astype(np.int64)
    t0 = A[:, 0][A[:, 0] > 0].min()
    flags = A[:, 7] & 0xFFFFFFFF
    ran = (A[:, 0] > 0)
    skipped = ran & ((flags & 1) == 1)
    full = ran & ~skipped
    print(f"CTAs {nA}: ran {ran.sum()}, skipped {skipped.sum()}, full {full.sum()}")
    F = A[full]
    ph = {"mask": F[:, 1] - F[:, 0], "p_wait": F[:, 2] - F[:, 1], "q_after_p": F[:, 3] - F[:, 2],
          "reduce": F[:, 4] - F[:, 3], "publish": F[:, 5] - F[:, 4], "tail": F[:, 6] - F[:, 5],
          "life": F[:, 6] - F[:, 0]}
    for kx, v in ph.items():
        v = v[(v >= 0) & (v < 10**7)]
        print(f"  {kx:10s} ns  p10 {np.percentile(v, 10):7.0f}  p50 {np.percentile(v, 50):7.0f}  "
              f"p90 {np.percentile(v, 90):7.0f}  mean {v.mean():7.0f}")
    sk = A[skipped]
    print(f"  skipped life p50 {np.percentile(sk[:, 1] - sk[:, 0], 50) if len(sk) else 0:.0f} ns")
    end = A[ran, 6].max()
    print(f"k_row_stats span {(end - t0) / 1e3:.1f} us")
    # per position: first start / last end (grid z = position when B <= 32768)
    gx, gy = nch, min(B, 32768)
    for j in range(k + 1):
        blk = A[j * gx * gy:(j + 1) * gx * gy]
        r = blk[blk[:, 0] > 0]
        fu = r[(r[:, 7] & 1) == 0]
        print(f"  pos {j}: start {(r[:, 0].min() - t0) / 1e3:6.1f}..{(r[:, 0].max() - t0) / 1e3:6.1f} us, "
              f"end ..{(r[:, 6].max() - t0) / 1e3:6.1f} us, full {len(fu)}/{len(r)}")
    # concurrency: CTAs alive / waiting for data, sampled every 1 us
    ts = np.arange(t0, end, 1000)
    alive = np.array([((A[ran, 0] <= t) & (A[ran, 6] > t)).sum() for t in ts])
    loading = np.array([((F[:, 1] <= t) & (np.maximum(F[:, 2], F[:, 3]) > t)).sum() for t in ts])
    print("  alive CTAs per us (every 5th):", alive[::5].tolist())
    print("  loading CTAs per us (every 5th):", loading[::5].tolist())
    if len(S) and (S[:, 0] > 0).any():
        print(f"k_sample_req: start {(S[:, 0].min() - t0) / 1e3:.1f} us, wait done "
              f"{(S[:, 1].min() - t0) / 1e3:.1f}..{(S[:, 1].max() - t0) / 1e3:.1f}, end "
              f"{(S[:, 2].min() - t0) / 1e3:.1f}..{(S[:, 2].max() - t0) / 1e3:.1f} us; per-CTA "
              f"p50 {np.percentile(S[:, 2] - S[:, 1], 50) / 1e3:.1f} us")
        ok = (S[:, 3] > 0) & (S[:, 4] > 0) & (S[:, 5] > 0)
        Q = S[ok]
        for nm, a_, b_ in (("first unit", 1, 3), ("stream rest", 3, 4), ("block search", 4, 5),
                           ("level 3 + outputs", 5, 2)):
            v = (Q[:, b_] - Q[:, a_]) / 1e3
            print(f"  sampler {nm:18s} p50 {np.percentile(v, 50):5.2f}  p90 {np.percentile(v, 90):5.2f} us")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--dtype", default="f32")
    ap.add_argument("--out", default="gpurun_out")
    ap.add_argument("--load", default=None, help="summarize a saved npz instead")
    a = ap.parse_args()
    if a.load:
        summarize(np.load(a.load))
        return
    c = CONFIGS[a.config]
    T = c["T"]
    dev = torch.device("cuda:0")
    dt = torch.float32 if a.dtype == "f32" else torch.bfloat16
    bs = [make_batch_torch(c["V"], c["k"], c["B"], T, c["kappa"], c["seed"] + i, dev, a.dtype)
          for i in range(4)]
    pl = sd.plan(c["B"], c["k"], c["V"], T, dt)
    nA = pl["ctas"]
    nch = nA // (c["B"] * (c["k"] + 1))          # grid x extent (padded chunks with clusters)
    buf = torch.zeros((nA + c["B"]) * 8, dtype=torch.int64, device=dev)
    for i in range(6):
        b = bs[i % 4]
        sd.verify(b["p"], b["q"] if T > 0 else None, b["ids"], T, seed=1, round=i)
    torch.cuda.synchronize()
    L = _lib.load()
    L.sd_debug_trace(ctypes.c_void_p(buf.data_ptr()))
    b = bs[1]
    out = sd.verify(b["p"], b["q"] if T > 0 else None, b["ids"], T, seed=1, round=99)
    torch.cuda.synchronize()
    L.sd_debug_trace(None)
    d = {"tr": buf.cpu().numpy().reshape(-1, 8), "nA": nA, "B": c["B"], "k": c["k"], "nch": nch,
         "L": out[0].cpu().numpy()}
    np.savez(os.path.join(a.out, f"rtrace_{a.config}_{a.dtype}.npz"), **d)
    print("mean L", float(out[0].float().mean()), "plan", pl)
    summarize(d)


if __name__ == "__main__":
    main()
