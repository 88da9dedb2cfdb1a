"""The fused cold-pick kernel (k_ffn_cold.cu) against the oracle: drain + gather +
swap-AB SwiGLU expert + forward into the home pools in one launch, for picks whose queues hold
<= 128 legs. Routing is given (round-robin experts, random weights) so every queue has an exact,
chosen size: ragged (17, 75), one token, the 128 maximum, 64 experts in one launch.

Integer results are exact (drained counts, the drained legs = the ring's FIFO prefix, every
token merged once); each pool row the kernel stored is compared, all columns, with the float64
oracle recomputing it from the GPU's own x (floored 2e-2; row-L2 mean 1e-3, max 4e-3, reading c13); the
merge is bit-exact given the pool; and the four-kernel path (AMOE_COLD=0) agrees within two
bf16 rounding steps (the stream-K split sums fp32 partials in another order)."""
import os

import numpy as np
import pytest
import torch

from oracle import numerics as nx
from parity_util import Problem, TOL, dev_tensor, floored_err, to_np

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    from paper_2505_08944_b200 import build
    build.build()


def _routing(T, E, K, seed):
    t = np.arange(T)[:, None]
    idx = ((t * K + np.arange(K)[None, :]) % E).astype(np.int32)      # K distinct experts per token
    w = np.random.default_rng(seed).random((T, K)).astype(np.float32) + 0.1
    w /= w.sum(1, keepdims=True)
    return idx, w.astype(np.float32)


def _run(P, idx, w, cold, hint):
    from paper_2505_08944_b200 import amoe
    old = os.environ.get("AMOE_COLD")
    os.environ["AMOE_COLD"] = "1" if cold else "0"
    try:
        ctx = P.make_ctx()
        ctx.set_exec_log(1 << 22)
        slots = torch.arange(P.T, dtype=torch.int32, device="cuda")
        ctx.token_init(slots, dev_tensor(P.h0[0], "bf16"), 0)
        ctx.enqueue(0, slots, topk_idx=torch.from_numpy(idx).cuda(), topk_w=torch.from_numpy(w).cuda())
        torch.cuda.synchronize()
        st = ctx.state()
        x0, h0 = to_np(st["x"]).copy(), to_np(st["h"]).copy()
        gb = amoe.GroupBuffers(ctx, P.E * 128 + 256).set_queues([(0, e) for e in range(P.E)], max_rows_hint=hint)
        l0 = ctx.launch_count()
        ctx.rebatch_ffn_forward(gb)
        launches = ctx.launch_count() - l0
        torch.cuda.synchronize()
        ctx.check()
        pool = to_np(ctx.state()["pool"]).copy()
        log = ctx.read_exec_log()
        ctx.combine(retire_pass=1)
        torch.cuda.synchronize()
        ctx.check()
        st = ctx.state()
        return dict(ctx=ctx, gb=gb, x0=x0, h0=h0, pool=pool, log=log, launches=launches,
                    h=to_np(st["h"]), merged=int(st["stats"][0]), legs=int(st["stats"][2]),
                    w=st["tok_w"].cpu().numpy())
    finally:
        if old is None:
            os.environ.pop("AMOE_COLD", None)
        else:
            os.environ["AMOE_COLD"] = old


@pytest.mark.parametrize("d,ff,E,K,T", [
    (512, 1024, 8, 2, 300),        # 75 legs per expert
    (256, 256, 8, 2, 68),          # small widths, 17 legs per expert (grid limited to the work)
    (2048, 1408, 8, 1, 1024),      # DeepSeek-shaped, 8 experts at the 128-leg maximum
    (2048, 1408, 1, 1, 1),         # one DeepSeek expert, one token
    (2048, 1408, 64, 6, 512),      # 64 DeepSeek experts in one launch, 48 legs each
    (4096, 14336, 1, 1, 100),      # one Mixtral expert, 100 tokens
])
def test_cold_kernel_matches_oracle(d, ff, E, K, T):
    P = Problem(L=1, E=E, K=K, S=0, d=d, ff=ff, T=T, seed=80 + E + K, n_tab=1)
    idx, w = _routing(T, E, K, 80 + T)
    hist = np.bincount(idx.ravel(), minlength=E)
    hint = int(hist.max())
    assert hint <= 128
    r = _run(P, idx, w, True, hint)
    assert r["launches"] == 1                                   # drain..forward in one launch
    n, off, start = r["gb"].info()
    assert n.tolist() == hist.tolist() and np.all(start == 0)
    assert r["legs"] == T * K and r["merged"] == T
    q2e = {r["ctx"].local_queue(e): e for e in range(E)}
    assert len(r["log"]) == E
    for (_, q, st0, legs) in r["log"]:
        e = q2e[q]
        assert st0 == 0 and len(legs) == hist[e]
        sl = np.array([g[0] for g in legs])
        ks = np.array([g[1] for g in legs])
        assert np.all(idx[sl, ks] == e)                          # every drained leg routed here
        ref = nx.expert_ffn(r["x0"][sl], *P.W[(0, e)])
        got = r["pool"][sl, ks]
        assert floored_err(got, ref) <= TOL["bf16"], (e, floored_err(got, ref))
        rl2 = np.linalg.norm(got - ref, axis=1) / np.maximum(np.linalg.norm(ref, axis=1), 1e-30)
        assert rl2.mean() <= 1e-3 and rl2.max() <= 4e-3, (e, rl2.mean(), rl2.max())   # reading c13
    assert np.array_equal(r["h"], nx.combine(r["h0"], r["w"], r["pool"][:, :K], None, "bf16"))
    # the four-kernel path on the same legs: two valid fp32 summation orders
    r0 = _run(P, idx, w, False, hint)
    assert r0["launches"] > 1
    assert floored_err(r["pool"], r0["pool"]) <= 2.0 ** -6


def test_cold_picks_inside_amoe_run_match_oracle(monkeypatch):
    """amoe_run takes the fused cold path for picks whose queues are all <= 128 deep: a spread
    start (tokens admitted at every layer) on the tiny widths, 2 passes, Algorithm 1 grouped and
    single-queue MTFS; every drain replayed through the oracle's µ-queues; h vs the oracle run."""
    from oracle import drivers
    from parity_util import ROW_L2, host_values, replay_exec_log, row_l2_err
    monkeypatch.setenv("AMOE_COLD", "1")
    P = Problem(L=2, E=8, K=2, S=0, d=256, ff=512, T=256, seed=90)
    for policy, grouped in (("defrag", True), ("mtfs", False)):
        ctx = P.make_ctx(max_batch=96)
        ctx.set_exec_log(1 << 22)
        ctx.profile_enable(True)
        slots = torch.arange(P.T, dtype=torch.int32, device="cuda")
        ctx.token_init(slots, dev_tensor(P.h0[0], "bf16"), 0)
        ctx.enqueue(0, slots, logits=torch.from_numpy(np.ascontiguousarray(P.tables[0][0, 0])).cuda())
        stats = ctx.run(retire_pass=2, policy=policy, grouped=grouped)
        torch.cuda.synchronize()
        ctx.check()
        prof = ctx.profile_read()
        assert prof["ffn_cold"][1] == stats["picks"] > 0           # every pick took the cold path
        log = ctx.read_exec_log()
        assert max(len(x[3]) for x in log) <= 96
        replay_exec_log(P.L, P.E, P.K, 0, 1, P.T, P.logits, 2, [log], [{ctx.local_queue(e): e for e in range(P.E)}])
        W, _ = P.oracle_weights()
        ref, _ = drivers.sync_run(host_values(P.h0[0], "bf16"), P.logits, W, P.K, n_passes=2)
        h = to_np(ctx.state()["h"])
        assert floored_err(h, ref) <= TOL["bf16"]
        assert row_l2_err(h, ref) <= ROW_L2["bf16"]
        ctx.close()


def test_execute_cold_explicit_drain_and_head_check():
    """amoe_execute_cold with the drain made explicit: two enqueue rounds on one queue, the
    second executed from ring position 37 (the head after draining 37 of the first 60 legs),
    leaves the other 23 + the new legs queued; a start that is not the head latches fault 12."""
    from paper_2505_08944_b200 import amoe
    from paper_2505_08944_b200.amoe import AmoeError
    P = Problem(L=1, E=1, K=1, S=0, d=256, ff=512, T=120, seed=5, n_tab=1)
    ctx = P.make_ctx()
    slots = torch.arange(P.T, dtype=torch.int32, device="cuda")
    ctx.token_init(slots, dev_tensor(P.h0[0], "bf16"), 0)
    one = torch.ones(60, 1, device="cuda")
    zero = torch.zeros(60, 1, dtype=torch.int32, device="cuda")
    ctx.enqueue(0, slots[:60], topk_idx=zero, topk_w=one)
    gb = amoe.GroupBuffers(ctx, 512).set_queues([(0, 0)])
    ctx.execute_cold(gb, [0], [37])
    torch.cuda.synchronize()
    ctx.check()
    assert ctx.queue_depths()[0, 0] == 23
    ctx.enqueue(0, slots[60:], topk_idx=zero, topk_w=one)
    ctx.execute_cold(gb, [37], [83])
    torch.cuda.synchronize()
    ctx.check()
    assert ctx.queue_depths()[0, 0] == 0
    st = ctx.state()
    assert int(st["stats"][2]) == 120
    x0 = to_np(st["x"])
    W = P.W[(0, 0)]
    pool = to_np(st["pool"])[:, 0]
    ref = nx.expert_ffn(x0, *W)
    assert floored_err(pool, ref) <= TOL["bf16"]
    ctx.combine(retire_pass=1)
    torch.cuda.synchronize()
    ctx.check()
    assert int(ctx.state()["stats"][0]) == 120          # every token merged exactly once
    # wrong start: the head is 120 now
    ctx.token_init(slots[:4], dev_tensor(P.h0[0][:4], "bf16"), 0)
    ctx.enqueue(0, slots[:4], topk_idx=zero[:4], topk_w=one[:4])
    ctx.execute_cold(gb, [119], [4])
    with pytest.raises(AmoeError) as ei:
        ctx.check()
    assert ei.value.info[:4] == [12, 0, 119, 120]


def test_execute_cold_ragged_with_empty_queue_and_maximum():
    """One fused cold launch over three DeepSeek-shaped queues holding 0, 5 and the 128-leg
    maximum: the empty queue drains nothing and stores nothing, the others match the oracle row
    for row, and the heads advance by exactly the drained counts."""
    from paper_2505_08944_b200 import amoe
    E, T = 3, 133
    P = Problem(L=1, E=E, K=1, S=0, d=2048, ff=1408, T=T, seed=19, n_tab=1)
    ctx = P.make_ctx()
    slots = torch.arange(T, dtype=torch.int32, device="cuda")
    ctx.token_init(slots, dev_tensor(P.h0[0], "bf16"), 0)
    idx = np.array([1] * 5 + [2] * 128, dtype=np.int32).reshape(T, 1)
    ctx.enqueue(0, slots, topk_idx=torch.from_numpy(idx).cuda(), topk_w=torch.ones(T, 1, device="cuda"))
    gb = amoe.GroupBuffers(ctx, 3 * 128 + 256).set_queues([(0, 0), (0, 1), (0, 2)])
    ctx.execute_cold(gb, [0, 0, 0], [0, 5, 128])
    torch.cuda.synchronize()
    ctx.check()
    n, _, start = gb.info()
    assert n.tolist() == [0, 5, 128] and start.tolist() == [0, 0, 0]
    assert ctx.queue_depths()[0].tolist()[:3] == [0, 0, 0]
    st = ctx.state()
    assert int(st["stats"][2]) == 133
    x0, pool = to_np(st["x"]), to_np(st["pool"])[:, 0]
    for e, rows in ((1, np.arange(5)), (2, np.arange(5, T))):
        ref = nx.expert_ffn(x0[rows], *P.W[(0, e)])
        assert floored_err(pool[rows], ref) <= TOL["bf16"], e
