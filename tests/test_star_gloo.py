"""The star's host protocol across processes, CPU only: a 1 -> 2 star over
torch.distributed gloo, three processes.  The draft (rank 0) runs the star's own FIFO scheduler
(sd_sched_*: Q_in) and ships ids + q rows for each (verifier, slot) round; each verifier
verifies with the CPU oracle (the GPU's stand-in here) on its own target rows and sends
(accept lengths, tokens) back; the draft polls completions, queues them in completion order and
serves FIFO, two slots per verifier (double buffering).  Checked: every round's result equals the
draft's own recomputation (the target rows are regenerated from shared seeds), the FIFO pops
follow completion order, every (verifier, slot, round) completes once, and the scheduler's
accounting (rounds, busy intervals) matches."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

V, K, B, SLOTS, ROUNDS, T = 257, 3, 4, 2, 4, 1.0


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _batch(v, s, r):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    from workload import make_batch
    return make_batch(V=V, k=K, B=B, T=T, kappa=30.0, seed=10_000 * v + 100 * s + r)


def _worker(rank, world, port, q):
    dbg = os.environ.get("STAR_GLOO_DEBUG")
    import sys
    import time
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    try:
        if rank == 0:
            from paper_2601_21622_b200 import star
            sc = star.Scheduler(world - 1, K)
            import queue
            import threading
            done_q = queue.Queue()
            order_done, popped, results = [], [], {}
            t0 = time.perf_counter()
            now = lambda: 1000.0 * (time.perf_counter() - t0)          # noqa: E731

            def submit(v, s, r):
                d = _batch(v, s, r)
                a = now()
                ids = torch.from_numpy(d["ids"])
                qq = torch.from_numpy(d["q"])
                if dbg:
                    print("draft submit", v, s, r, flush=True)
                dist.send(torch.tensor([s, r], dtype=torch.int64), dst=v)
                dist.send(ids, dst=v)
                dist.send(qq, dst=v)
                sc.service(v, a, now())
                L = torch.empty(B, dtype=torch.int32)
                tok = torch.empty(B, K + 1, dtype=torch.int32)
                w1 = dist.irecv(L, src=v, tag=2 * s)
                w2 = dist.irecv(tok, src=v, tag=2 * s + 1)

                def waiter():                  # the receiver thread of P:276-279
                    w1.wait()
                    w2.wait()
                    done_q.put((v, s, r, L, tok))
                threading.Thread(target=waiter, daemon=True).start()

            for s in range(SLOTS):
                for v in range(1, world):
                    submit(v, s, 0)
            total = (world - 1) * SLOTS * ROUNDS
            while len(popped) < total:
                while not done_q.empty():      # completed returns enter Q_in in completion order
                    v, s, r, L, tok = done_q.get()
                    sc.push(v, s, r, now())
                    order_done.append((v, s, r))
                    results[(v, s, r)] = (L.numpy().copy(), tok.numpy().copy())
                got = sc.pop(now())
                if got is None:
                    time.sleep(0.001)
                    continue
                popped.append(got)
                v, s, r = got
                sc.observe(v, 1.0, results[(v, s, r)][0])
                if r + 1 < ROUNDS:
                    submit(v, s, r + 1)
            for v in range(1, world):
                dist.send(torch.tensor([-1, -1], dtype=torch.int64), dst=v)
            # recompute every round on the draft (target rows regenerated from the shared seeds)
            bad = 0
            for (v, s, r), (L, tok) in results.items():
                d = _batch(v, s, r)
                rL, rtok, _ = oracle.verify(d["p"], d["q"], d["ids"], T, seed=5, round=r,
                                            rid_base=(v << 32) + s * B)
                bad += int(not (np.array_equal(rL, L) and np.array_equal(rtok, tok)))
            st = sc.stats()
            q.put(("draft", popped == order_done, sorted(popped), bad, st["rounds"],
                   st["busy_fraction"]))
        else:
            while True:
                hdr = torch.empty(2, dtype=torch.int64)
                dist.recv(hdr, src=0)
                s, r = int(hdr[0]), int(hdr[1])
                if s < 0:
                    break
                ids = torch.empty(B, K, dtype=torch.int32)
                qq = torch.empty(B, K, V, dtype=torch.float32)
                dist.recv(ids, src=0)
                dist.recv(qq, src=0)
                if dbg:
                    print("verifier", rank, "got", s, r, flush=True)
                d = _batch(rank, s, r)                 # this verifier's own target rows
                L, tok, _ = oracle.verify(d["p"], qq.numpy(), ids.numpy(), T, seed=5, round=r,
                                          rid_base=(rank << 32) + s * B)
                dist.send(torch.from_numpy(L), dst=0, tag=2 * s)
                dist.send(torch.from_numpy(tok), dst=0, tag=2 * s + 1)
            q.put(("verifier", rank))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_gloo_star_protocol_three_processes():
    world = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    draft = next(r for r in res if r[0] == "draft")
    _, fifo_ok, popped, bad, rounds, busy = draft
    assert fifo_ok                                    # served in completion (Q_in) order
    want = sorted((v, s, r) for v in (1, 2) for s in range(SLOTS) for r in range(ROUNDS))
    assert popped == want                             # every round exactly once
    assert bad == 0                                   # results crossed processes intact
    assert rounds == len(want) and 0.0 < busy <= 1.0
