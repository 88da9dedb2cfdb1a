"""N>1 host logic on CPU: two gloo processes exercise the partition and the max-over-ranks timing
reduction bench.py uses (the data path itself has no collective; its kernels are covered by the
loopback-peer GPU test)."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), WORLD_SIZE=str(world), RANK=str(rank),
                      LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2505_08944_b200 import dist as D
    G, r, lr = D.env()
    assert (G, r, lr) == (world, rank, rank)
    ms, counts = D.reduce_timing(10.0 * (rank + 1), [100 + rank, 7])
    D.barrier()
    toks = list(D.token_range(rank, 16))
    hosted = D.hosted_experts(8, 2, world, rank)
    per_rank = D.gather_values([0.25 * rank, rank + 3])
    assert per_rank == [[0.25 * r, r + 3.0] for r in range(world)]
    q.put((rank, ms, counts, toks, hosted))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_partition_and_timing(world):
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ms, counts, toks, hosted in res:
        assert ms == 10.0 * world                              # max over ranks
        assert counts == [sum(100 + r for r in range(world)), 7 * world]
        assert hosted[-2:] == [8, 9]                           # shared experts on every rank
    all_toks = sorted(t for r in res for t in r[3])
    assert all_toks == list(range(16 * world))                 # every token homed exactly once
    routed = sorted(e for r in res for e in r[4] if e < 8)
    assert routed == list(range(8))                            # every expert owned exactly once
