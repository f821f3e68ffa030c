"""Star round scheduler on one GPU vs the closed forms of Sec. 4.1 (PAPER.md
Eqs. 7-10).

Loopback transport: this process is the draft and N virtual verifiers.  The draft's per-round
service time S(d) (Eq. 5) is a device spin of S ms on the draft stream between draft_begin() and
draft_end(); the verifier's target forward is a device spin of Z ms (`target_ms`, sd_star_config)
on the pair's stream before the real verify kernels, so the return time is Z(d) = Z + t_verify
(Eq. 6).  The draft is work-conserving (Alg. 1): whichever verifier comes back first
is served next.  Reports the measured busy fraction / idle gaps (device-clock CUDA events, the
library's own sd_star_stats) beside predicted(N, S, Z).

  python tools/star_bench.py [--S 2 --Z 6 --N 1 2 3 4 7 --slots 1 2 --rounds 40]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_21622_b200 import star  # noqa: E402


def sleep_cycles_per_ms() -> float:
    """Calibrate torch.cuda._sleep (SM clock cycles) against CUDA events."""
    torch.cuda._sleep(1_000_000)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 20_000_000
    a.record()
    torch.cuda._sleep(n)
    b.record()
    b.synchronize()
    return n / a.elapsed_time(b)


def run(N: int, slots: int, S: float, Z: float, rounds: int, cyc_per_ms: float,
        B: int, k: int, V: int) -> dict:
    dev = torch.device("cuda:0")
    h = star.Star(0, N + 1, B, k, V, 1.0, seed=5, n_slots=slots, device=dev,
                  transport="loopback", target_ms=Z)
    g = torch.Generator(device=dev).manual_seed(1)
    p = torch.randn(B, k + 1, V, device=dev, generator=g) * 3
    q = torch.randn(B, k, V, device=dev, generator=g) * 3
    ids = torch.randint(0, V, (B, k), device=dev, dtype=torch.int32, generator=g)
    bufs = {(v, s): (torch.empty(B, dtype=torch.int32, device=dev),
                     torch.empty(B, k + 1, dtype=torch.int32, device=dev))
            for v in range(1, N + 1) for s in range(slots)}
    cyc = int(S * cyc_per_ms)
    nxt = {}

    def draft_and_submit(v, s):
        r = nxt.get((v, s), 0)
        h.draft_begin()
        torch.cuda._sleep(cyc)                 # S(d): the draft's k forward passes
        h.draft_end()
        L, tok = bufs[(v, s)]
        h.submit(v, s, r, ids, q, L, tok, request_id_base=(v << 32) + (s << 24), p=p)
        nxt[(v, s)] = r + 1

    total = rounds * N * slots
    for s in range(slots):
        for v in range(1, N + 1):
            draft_and_submit(v, s)
    served = N * slots
    done = 0
    while done < total:
        got = h.poll(timeout_us=30_000_000)
        if got is None:
            raise RuntimeError("no return within 30 s")
        v, s, _ = got
        done += 1
        if served < total:
            draft_and_submit(v, s)
            served += 1
    torch.cuda.synchronize()
    st = h.stats()
    h.close()
    return st


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--S", type=float, default=2.0, help="draft service time per round, ms")
    ap.add_argument("--Z", type=float, default=6.0, help="target forward stand-in, ms")
    ap.add_argument("--N", type=int, nargs="+", default=[1, 2, 3, 4, 5, 7])
    ap.add_argument("--slots", type=int, nargs="+", default=[1, 2])
    ap.add_argument("--rounds", type=int, default=30, help="rounds per (verifier, slot)")
    ap.add_argument("--B", type=int, default=16)
    ap.add_argument("--k", type=int, default=5)
    ap.add_argument("--V", type=int, default=32000)
    a = ap.parse_args()
    cpm = sleep_cycles_per_ms()
    for slots in a.slots:
        for N in a.N:
            st = run(N, slots, a.S, a.Z, a.rounds, cpm, a.B, a.k, a.V)
            pred = star.predicted(N, a.S, a.Z)
            print(json.dumps({"N": N, "slots": slots, "S_ms": a.S, "Z_ms": a.Z,
                              "busy_fraction": round(st["busy_fraction"], 4),
                              "mean_idle_ms": round(st["mean_idle_ms"], 4),
                              "mean_wait_ms": round(st["mean_wait_ms"], 4),
                              "rounds": st["rounds"],
                              "predicted_1slot": {k: round(v, 4) for k, v in pred.items()}}),
                  flush=True)


if __name__ == "__main__":
    main()
