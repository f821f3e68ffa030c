"""Star exchange over NCCL, one process per GPU (Alg. 1).

  python -m torch.distributed.run --nnodes=1 --nproc-per-node 1+N --master-addr 127.0.0.1 \
      --master-port 29511 tools/star_demo.py --rounds 50

Rank 0 is the draft: it "drafts" (synthetic q rows + ids, with --draft-ms of device work to
stand in for M_q's S(d)), submits each round to the verifier whose return came back first
(FIFO over Q_in) and reports the scheduler stats.  Ranks 1..N verify with the
sm_100a kernels and send back (L, tokens).  Needs >= 2 GPUs on one node.
"""
import argparse
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_21622_b200 import star  # noqa: E402
from workload import make_batch_torch  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rounds", type=int, default=50)
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--k", type=int, default=4)
    ap.add_argument("--vocab", type=int, default=32000)
    ap.add_argument("--slots", type=int, default=2)
    ap.add_argument("--temperature", type=float, default=1.0)
    ap.add_argument("--draft-ms", type=float, default=2.0)
    a = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("gloo")                     # host-side handshake only
    ids = star.exchange_ids(rank, world)
    h = star.Star(rank, world, a.batch, a.k, a.vocab, a.temperature, seed=5, n_slots=a.slots,
                  device=dev, ids=ids)
    B, k, V = a.batch, a.k, a.vocab
    per_stream = a.rounds
    if rank == 0:
        bufs = {}
        spin = torch.empty(1 << 20, device=dev)

        def draft_and_submit(v, s, r):
            h.draft_begin()
            bt = make_batch_torch(V, k, B, a.temperature, 30.0, seed=r * 1000 + v * 10 + s, device=dev)
            t_end = torch.cuda.Event(enable_timing=True)
            t0 = torch.cuda.Event(enable_timing=True)
            t0.record()
            while True:                                  # stand-in for M_q's S(d)
                spin.mul_(1.0001)
                t_end.record()
                t_end.synchronize()
                if t0.elapsed_time(t_end) >= a.draft_ms:
                    break
            h.draft_end()
            L = torch.empty(B, dtype=torch.int32, device=dev)
            tok = torch.empty(B, k + 1, dtype=torch.int32, device=dev)
            h.submit(v, s, r, bt["ids"], bt["q"], L, tok, request_id_base=(v << 32) + s * B)
            bufs[(v, s)] = (bt, L, tok)

        for s in range(a.slots):
            for v in range(1, world):
                draft_and_submit(v, s, 0)
        done, emitted = 0, 0
        total = (world - 1) * a.slots * per_stream
        while done < total:
            got = h.poll(timeout_us=30_000_000)
            if got is None:
                raise SystemExit("timeout waiting for a verifier")
            v, s, r = got
            _, L, _ = bufs[(v, s)]
            emitted += int((L + 1).sum())
            done += 1
            if r + 1 < per_stream:
                draft_and_submit(v, s, r + 1)
        st = h.stats()
        st.update({"verifiers": world - 1, "slots": a.slots, "tokens_emitted": emitted})
        print(json.dumps(st), flush=True)
    else:
        for r in range(per_stream):
            for s in range(a.slots):
                # the verifier's own target logits for this round (synthetic, same recipe)
                bt = make_batch_torch(V, k, B, a.temperature, 30.0, seed=r * 1000 + rank * 10 + s,
                                      device=dev)
                L = torch.empty(B, dtype=torch.int32, device=dev)
                tok = torch.empty(B, k + 1, dtype=torch.int32, device=dev)
                h.serve(s, r, B, bt["p"], L, tok, request_id_base=(rank << 32) + s * B)
        torch.cuda.synchronize()
    h.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
