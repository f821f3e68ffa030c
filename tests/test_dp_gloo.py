"""N>1 host logic on CPU with a world_size-2 gloo group (SURVEY §8 e, f): the bench's job
aggregation (max time over ranks, summed units), disjoint per-rank Philox request ranges, and
the star handshake (communicator ids broadcast from the draft rank)."""
import os
import socket
import sys

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    from paper_2601_21622_b200 import dp, star
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        # rank r "ran" 10 + r ms and processed 100 * (r + 1) tokens
        mx, sm = dp.reduce_max_sum([10.0 + rank, 1.0], [100.0 * (rank + 1)])
        ids = star.exchange_ids(rank, world)
        q.put((rank, mx, sm, dp.request_id_base(rank), ids))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_gloo_world2_aggregation_and_handshake():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, mx, sm, rid, ids in res:
        assert mx == [11.0, 1.0]                 # MAX over ranks: the job's device time
        assert sm == [300.0]                     # SUM: units processed by all ranks
        assert rid == rank << 32
        assert len(ids) == 2 * 128 * (world - 1)   # one id per direction per (0, v) pair
    assert res[0][4] == res[1][4]                # every rank holds the draft's ids
    # disjoint 2^32-request Philox ranges
    assert res[1][3] - res[0][3] == 1 << 32


def test_request_id_base_single_process():
    from paper_2601_21622_b200 import dp
    assert dp.request_id_base(0) == 0
    assert dp.request_id_base(7) == 7 << 32
    with pytest.raises(ValueError):
        dp.request_id_base(-1)
    mx, sm = dp.reduce_max_sum([3.0], [4.0])
    assert mx == [3.0] and sm == [4.0]
