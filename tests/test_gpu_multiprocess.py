"""The multi-process path of bench.py / amoe_run on one GPU: two ranks in two processes (gloo
process group for setup), workspaces peer-mapped with CUDA IPC handles exchanged through the
group (paper_2505_08944_b200.dist.peer_workspace), experts owned e mod 2, each rank running the
native scheduler loop. Legs cross processes through IPC-mapped rings with system-scope atomics —
the same code path as NVLink peers on an 8-GPU box. Result must equal one rank, bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_main(rank, world, port, T, q):
    try:
        import sys
        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        sys.path.insert(0, root)
        sys.path.insert(0, os.path.join(root, "tests"))
        import torch.distributed as dist
        # bitwise vs one rank: unsplit FFN path only (the cold kernel's split order depends on
        # the pick's shape)
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), AMOE_COLD="0")
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        from paper_2505_08944_b200 import amoe, dist as D
        from parity_util import Problem, dev_tensor, to_np
        P = Problem(L=2, E=8, K=2, S=0, d=256, ff=512, T=T, G=world, seed=21)
        cfg = amoe.make_config(P.L, P.E, P.K, P.S, P.d, P.ff, T, G=world, rank=rank)
        ws, ptrs = D.peer_workspace(amoe.workspace_bytes(cfg), torch.device("cuda", 0), method="ipc")
        ctx = amoe.Context(cfg, workspace=ws)
        ctx.import_peers(ptrs)
        for l in range(P.L):
            for e in D.hosted_experts(P.E, P.S, world, rank):
                ctx.set_expert(l, e, *P.Wd[(l, e)])
        ctx.set_router(torch.from_numpy(P.tables[rank]).cuda().contiguous())
        ctx.set_exec_log(1 << 22)
        torch.cuda.synchronize()
        dist.barrier()           # all workspaces created (zeroed) before any rank pushes legs
        slots = torch.arange(T, dtype=torch.int32, device="cuda")
        ctx.token_init(slots, dev_tensor(P.h0[rank], "bf16"), 0)
        ctx.enqueue(0, slots, logits=torch.from_numpy(np.ascontiguousarray(P.tables[rank][0, 0])).cuda())
        dist.barrier()
        stats = ctx.run(retire_pass=2)
        torch.cuda.synchronize()
        ctx.check()
        q2e = {ctx.local_queue(e): e for e in D.hosted_experts(P.E, P.S, world, rank)}
        q.put((rank, to_np(ctx.state()["h"]), stats, int(ctx.state()["stats"][3]), ctx.read_exec_log(), q2e))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - surfaced by the parent
        import traceback
        q.put((rank, None, traceback.format_exc(), 0, None, None))


def test_two_processes_one_gpu_match_single_rank(monkeypatch):
    monkeypatch.setenv("AMOE_COLD", "0")
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required")
    world, T = 2, 128
    ctx_mp = mp.get_context("spawn")
    q = ctx_mp.Queue()
    port = _port()
    procs = [ctx_mp.Process(target=_rank_main, args=(r, world, port, T, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, h, stats, remote, log, q2e = q.get(timeout=300)
        assert h is not None, stats
        res[r] = (h, stats, remote, log, q2e)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert sum(v[1]["token_layers"] for v in res.values()) == world * T * 2 * 2
    assert all(v[2] > 0 for v in res.values())              # legs crossed processes
    from parity_util import Problem, dev_tensor, to_np
    P = Problem(L=2, E=8, K=2, S=0, d=256, ff=512, T=T, G=world, seed=21)
    P1 = Problem(L=2, E=8, K=2, S=0, d=256, ff=512, T=world * T, G=1, seed=21)
    P1.tables = [np.concatenate(P.tables, axis=2)]
    P1.h0 = [np.concatenate(P.h0)]
    c1 = P1.make_ctx()
    slots = torch.arange(world * T, dtype=torch.int32, device="cuda")
    c1.token_init(slots, dev_tensor(P1.h0[0], "bf16"), 0)
    c1.enqueue(0, slots, logits=torch.from_numpy(np.ascontiguousarray(P1.tables[0][0, 0])).cuda())
    c1.run(retire_pass=2)
    torch.cuda.synchronize()
    h1 = to_np(c1.state()["h"])
    h = np.concatenate([res[0][0], res[1][0]])
    assert np.array_equal(h, h1)
    # against the oracle: every drain of both processes replayed through Box(G=2), per-rank leg
    # counts = the legs routed to its experts, h vs the synchronous run (reading c13)
    from oracle import drivers
    from parity_util import TOL, floored_err, host_values, replay_exec_log
    _, counts = replay_exec_log(P.L, P.E, P.K, P.S, world, T, P.logits, 2, [res[r][3] for r in range(world)],
                                [res[r][4] for r in range(world)])
    for r in range(world):
        assert res[r][1]["legs"] == sum(v for k, v in counts.items() if k[0] == r)
    W, SH = P.oracle_weights()
    ref, _ = drivers.sync_run(np.concatenate([host_values(x, "bf16") for x in P.h0]), P.logits, W, P.K,
                              n_passes=2, shared=SH)
    assert floored_err(h, ref) <= TOL["bf16"]
