"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times (grouped
Algorithm-1 pick over all experts of a layer, CTA-pair tcgen05 kernels): one Mixtral-shaped layer
(E=8, top-2, d=4096, ff=14336) with 16384 tokens in flight. The oracle recomputes sampled rows one
by one (float64); integer results are checked in full."""
import os

import numpy as np
import pytest
import torch

from oracle import numerics as nx
from parity_util import ROW_L2, Problem, TOL, dev_tensor, floored_err, host_values, row_l2_err, to_np

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    from paper_2505_08944_b200 import build
    build.build()


def _run_layer(P, ctx):
    from paper_2505_08944_b200 import amoe
    slots = torch.arange(P.T, dtype=torch.int32, device="cuda")
    ctx.token_init(slots, dev_tensor(P.h0[0], P.dtype), 0)
    ctx.enqueue(0, slots, logits=torch.from_numpy(np.ascontiguousarray(P.tables[0][0, 0])).cuda())
    gb = amoe.GroupBuffers(ctx, P.T * (P.K + P.S) + 128 * (P.E + P.S))
    gb.set_queues([(0, e) for e in range(P.E + P.S)])
    ctx.rebatch(gb)
    ctx.expert_ffn(gb)
    torch.cuda.synchronize()
    ctx.check()
    return gb


@pytest.mark.parametrize("d,ff,T", [(512, 1024, 2048), (2048, 1408, 4096)])
def test_pair_kernel_matches_oracle_and_1cta(d, ff, T):
    """CTA-pair (cta_group::2, M=256) kernels vs the oracle, and vs the 1-CTA kernels."""
    P = Problem(L=1, E=8, K=2, S=0, d=d, ff=ff, T=T, seed=11)
    os.environ["AMOE_FFN_1CTA"] = "0"
    try:
        ctx = P.make_ctx()
        gb = _run_layer(P, ctx)
    finally:
        os.environ.pop("AMOE_FFN_1CTA")
    n, off, _ = gb.info()
    tile, out = to_np(gb.tile), to_np(gb.out)
    out_pair = out.copy()
    for i in range(P.E):
        rows = slice(off[i], off[i] + n[i])
        ref = nx.expert_ffn(tile[rows], *P.W[(0, i)])
        assert floored_err(out[rows], ref) <= TOL["bf16"]
        assert row_l2_err(out[rows], ref) <= 2e-3
    os.environ["AMOE_FFN_1CTA"] = "1"
    try:
        ctx2 = P.make_ctx()
        gb2 = _run_layer(P, ctx2)
    finally:
        os.environ.pop("AMOE_FFN_1CTA")
    out1, tile1 = to_np(gb2.out), to_np(gb2.tile)
    n1, off1, _ = gb2.info()
    meta0, meta1 = gb.meta.cpu().numpy(), gb2.meta.cpu().numpy()
    assert np.array_equal(n1, n)
    for i in range(P.E):
        rows, rows1 = slice(off[i], off[i] + n[i]), slice(off1[i], off1[i] + n1[i])
        e_pair = floored_err(out_pair[rows], nx.expert_ffn(tile[rows], *P.W[(0, i)]))
        e_one = floored_err(out1[rows1], nx.expert_ffn(tile1[rows1], *P.W[(0, i)]))
        # ring order inside a queue differs between runs (concurrent producers): align by leg
        k0 = meta0[rows, 0].astype(np.int64) * 16 + (meta0[rows, 1] & 0xFFFF)
        k1 = meta1[rows1, 0].astype(np.int64) * 16 + (meta1[rows1, 1] & 0xFFFF)
        o0, o1 = out_pair[rows][np.argsort(k0)], out1[rows1][np.argsort(k1)]
        assert np.array_equal(np.sort(k0), np.sort(k1))
        # each is within one bf16 ulp of the exact value; a stale-stage race would show up as a
        # large, localised difference
        assert e_pair <= 2.0 ** -7 and e_one <= 2.0 ** -7, (i, e_pair, e_one)
        assert floored_err(o1, o0) <= 2.0 ** -6


@pytest.mark.parametrize("pair", ["0", "1"])
def test_fused_forward_equals_separate_forward(pair):
    """amoe_expert_ffn_forward (rows stored into the home pools by the down-GEMM epilogue) gives
    the same pool rows and the same merged tokens, bit for bit, as expert_ffn + forward."""
    P = Problem(L=2, E=8, K=2, S=0, d=512, ff=1024, T=1024, seed=13)
    os.environ["AMOE_FFN_1CTA"] = "1" if pair == "0" else "0"
    try:
        res = []
        for fused in (False, True):
            ctx = P.make_ctx()
            from paper_2505_08944_b200 import amoe
            slots = torch.arange(P.T, dtype=torch.int32, device="cuda")
            ctx.token_init(slots, dev_tensor(P.h0[0], P.dtype), 0)
            ctx.enqueue(0, slots, logits=torch.from_numpy(np.ascontiguousarray(P.tables[0][0, 0])).cuda())
            gb = amoe.GroupBuffers(ctx, P.T * P.K + 128 * P.E).set_queues([(0, e) for e in range(P.E)])
            ctx.rebatch(gb)
            if fused:
                ctx.expert_ffn_forward(gb)
            else:
                ctx.expert_ffn(gb)
                ctx.forward(gb)
            torch.cuda.synchronize()
            ctx.check()
            pool = to_np(ctx.state()["pool"]).copy()
            ctx.combine(retire_pass=1)
            torch.cuda.synchronize()
            ctx.check()
            st = ctx.state()
            res.append((pool, to_np(st["h"]), int(st["stats"][0]), int(st["stats"][2])))
    finally:
        os.environ.pop("AMOE_FFN_1CTA")
    (p0, h0, m0, l0), (p1, h1, m1, l1) = res
    assert np.array_equal(p0, p1) and np.array_equal(h0, h1)
    assert m0 == m1 == P.T and l0 == l1 == P.T * P.K


@pytest.mark.parametrize("pair,d,S,T,how", [("0", 512, 0, 1000, "tma4"), ("1", 512, 0, 1000, "tma4"),
                                             ("1", 2048, 2, 1000, "tma4"), ("1", 512, 0, 1000, "cp"),
                                             ("1", 2048, 2, 1000, "cp"), ("1", 2048, 2, 3001, "cp"),
                                             ("1", 4096, 0, 2500, "cp")])
def test_fused_gather_equals_materialised_gather(pair, d, S, T, how):
    """amoe_rebatch_ffn_forward (gather inside the gate/up A load — TMA tile::gather4, or the
    producer warp's cp.async copies (AMOE_CP_GATHER=1) — legs read from the rings, forward inside the
    down epilogue) == rebatch + expert_ffn + forward, bitwise: same pool rows, same merged
    tokens, same counts; ragged queue tails and several M tiles per queue included."""
    ff = {512: 1024, 2048: 1408, 4096: 2048}[d]
    P = Problem(L=2, E=8, K=2, S=S, d=d, ff=ff, T=T, seed=15)
    os.environ["AMOE_FFN_1CTA"] = "1" if pair == "0" else "0"
    os.environ["AMOE_FUSED_GATHER" if how == "tma4" else "AMOE_CP_GATHER"] = "1"
    try:
        res = []
        for fused in (False, True):
            ctx = P.make_ctx()
            from paper_2505_08944_b200 import amoe
            slots = torch.arange(P.T, dtype=torch.int32, device="cuda")
            ctx.token_init(slots, dev_tensor(P.h0[0], P.dtype), 0)
            ctx.enqueue(0, slots, logits=torch.from_numpy(np.ascontiguousarray(P.tables[0][0, 0])).cuda())
            gb = amoe.GroupBuffers(ctx, P.T * (P.K + P.S) + 128 * (P.E + P.S))
            gb.set_queues([(0, e) for e in range(P.E + P.S)])
            if fused:
                ctx.rebatch_ffn_forward(gb)
            else:
                ctx.rebatch(gb)
                ctx.expert_ffn(gb)
                ctx.forward(gb)
            torch.cuda.synchronize()
            ctx.check()
            pool = to_np(ctx.state()["pool"]).copy()
            ctx.combine(retire_pass=1)
            torch.cuda.synchronize()
            ctx.check()
            st = ctx.state()
            res.append((pool, to_np(st["h"]), int(st["stats"][0])))
    finally:
        os.environ.pop("AMOE_FFN_1CTA")
        os.environ.pop("AMOE_FUSED_GATHER", None)
        os.environ.pop("AMOE_CP_GATHER", None)
    (p0, h0, m0), (p1, h1, m1) = res
    assert m0 == m1 == P.T
    assert np.array_equal(p0, p1) and np.array_equal(h0, h1)


@pytest.mark.parametrize("pair,d,ff,T", [("1", 2048, 1408, 40), ("0", 2048, 1408, 40), ("1", 4096, 2048, 100),
                                         ("1", 2048, 1408, 300)])
def test_split_k_cold_expert(pair, d, ff, T):
    """Cold experts (fewer output tiles than SMs) split K across CTAs with a fixed-order fp32
    reduction by the last arriving unit: outputs meet the oracle gate and stay within two bf16
    ulps of the unsplit kernels; the fused forward of split tiles returns every leg exactly once."""
    P = Problem(L=1, E=4, K=1, S=0, d=d, ff=ff, T=T, seed=16)
    outs = []
    os.environ["AMOE_FFN_1CTA"] = "1" if pair == "0" else "0"
    try:
        for split in ("1", "0"):
            os.environ["AMOE_SPLITK"] = split
            ctx = P.make_ctx()
            gb = _run_layer(P, ctx)
            n, off, _ = gb.info()
            outs.append((to_np(gb.tile), to_np(gb.out), gb.meta.cpu().numpy(), n, off))
            if split == "1":
                # separate forward + merge vs fused forward (split tiles) + merge: identical tokens
                ctx.forward(gb)
                ctx.combine(retire_pass=1)
                torch.cuda.synchronize()
                ctx.check()
                assert int(ctx.state()["stats"][0]) == P.T
                from paper_2505_08944_b200 import amoe
                c2 = P.make_ctx()
                slots = torch.arange(P.T, dtype=torch.int32, device="cuda")
                c2.token_init(slots, dev_tensor(P.h0[0], P.dtype), 0)
                c2.enqueue(0, slots, logits=torch.from_numpy(np.ascontiguousarray(P.tables[0][0, 0])).cuda())
                g2 = amoe.GroupBuffers(c2, P.T * P.K + 128 * P.E).set_queues([(0, e) for e in range(P.E)])
                c2.rebatch(g2)
                c2.expert_ffn_forward(g2)
                c2.combine(retire_pass=1)
                torch.cuda.synchronize()
                c2.check()
                assert int(c2.state()["stats"][0]) == P.T
                assert np.array_equal(to_np(c2.state()["h"]), to_np(ctx.state()["h"]))
    finally:
        os.environ.pop("AMOE_SPLITK", None)
        os.environ.pop("AMOE_FFN_1CTA", None)
    (t0, o0, m0, n, off), (t1, o1, m1, n1, off1) = outs
    for i in range(P.E):
        if n[i] == 0:
            continue
        r0, r1 = slice(off[i], off[i] + n[i]), slice(off1[i], off1[i] + n1[i])
        ref = nx.expert_ffn(t0[r0], *P.W[(0, i)])
        assert floored_err(o0[r0], ref) <= 2.0 ** -7, (i, floored_err(o0[r0], ref))
        k0, k1 = m0[r0, 0], m1[r1, 0]
        a0, a1 = o0[r0][np.argsort(k0)], o1[r1][np.argsort(k1)]
        assert floored_err(a0, a1) <= 2.0 ** -6


@pytest.mark.slow
@pytest.mark.parametrize("shape", ["mixtral", "deepseek"])
def test_layer_fullsize_every_m_tile(shape):
    """One full-size layer through the bench's own path: amoe_run (Algorithm-1 grouped pick ->
    amoe_rebatch_ffn_forward: drain, gather, CTA-pair tcgen05 gate/up + SwiGLU, down with the
    forward fused into its epilogue, dynamic tile schedule -> combine), 16384 tokens in flight.
    - Integer parity, in full: every drain is logged (checked mode) and replayed through the
      oracle's µ-queues (each leg routed there, taken once, FIFO-contiguous, router weight);
      drained counts = the router histogram.
    - Numerics, every M tile: from every execution, one random row out of every 128-row block
      of its drained legs (each CTA's half of every 256-row pair tile, ragged tails included),
      plus its last row, is recomputed by the float64 oracle from the GPU's own x and compared,
      all columns, with the row the fused epilogue stored into the home token pool (floored 2e-2;
      row-L2 mean <= 2e-3 (reading c13's diagnostic) and max <= 4e-3).
    - The merge of every token is bit-exact (teacher-forced on the GPU's pool and weights) and
      x_{l+1} is within one bf16 ulp of rmsnorm(h)."""
    from parity_util import replay_exec_log, ulp_err
    if shape == "mixtral":
        P = Problem(L=1, E=8, K=2, S=0, d=4096, ff=14336, T=16384, seed=12, n_tab=1)
    else:
        P = Problem(L=1, E=64, K=6, S=2, d=2048, ff=1408, T=16384, seed=13, n_tab=1)
    ctx = P.make_ctx()
    ctx.set_exec_log(64 << 20)
    slots = torch.arange(P.T, dtype=torch.int32, device="cuda")
    ctx.token_init(slots, dev_tensor(P.h0[0], P.dtype), 0)
    ctx.enqueue(0, slots, logits=torch.from_numpy(np.ascontiguousarray(P.tables[0][0, 0])).cuda())
    torch.cuda.synchronize()
    st = ctx.state()
    x0 = to_np(st["x"]).copy()
    h_before = to_np(st["h"]).copy()
    stats = ctx.run(retire_pass=1)
    torch.cuda.synchronize()
    ctx.check()
    assert stats["token_layers"] == P.T and stats["legs"] == P.T * (P.K + P.S)
    log = ctx.read_exec_log()
    q2e = {ctx.local_queue(e): e for e in range(P.E + P.S)}
    _, counts = replay_exec_log(P.L, P.E, P.K, P.S, 1, P.T, P.logits, 1, [log], [q2e])
    idx, _ = nx.route_topk(P.logits(0, 0), P.K)
    hist = np.concatenate([np.bincount(idx.ravel(), minlength=P.E), np.full(P.S, P.T)])
    assert [counts.get((0, 0, e, 0), 0) for e in range(P.E + P.S)] == hist.tolist()
    st = ctx.state()
    pool = to_np(st["pool"])
    g = np.random.default_rng(0)
    by_e = {}
    for (_, q, _, legs) in log:
        n = len(legs)
        picks = {n - 1} | {m0 + int(g.integers(0, min(128, n - m0))) for m0 in range(0, n, 128)}
        by_e.setdefault(q2e[q], []).extend((legs[i][0], legs[i][1]) for i in sorted(picks))
    checked = 0
    for e, rows in by_e.items():
        sl = np.array([r[0] for r in rows])
        ks = np.array([r[1] for r in rows])
        ref = nx.expert_ffn(x0[sl], *P.W[(0, e)])
        got = pool[sl, ks]
        assert floored_err(got, ref) <= TOL["bf16"], (e, floored_err(got, ref))
        rl2 = np.linalg.norm(got - ref, axis=1) / np.linalg.norm(ref, axis=1)
        # reading c13's diagnostic (mean row-L2 <= 2e-3): bf16 output rounding alone puts a row's
        # relative L2 error near 1e-3, so a mean over a few randomly sampled rows at 1e-3 (this
        # test's former gate, tighter than c13) fails by chance (1.07e-3 on expert 13 of a DeepSeek
        # layer, profiles/r02/fullsize_rowl2_flake.log)
        assert rl2.mean() <= ROW_L2["bf16"] and rl2.max() <= 4e-3, (e, rl2.mean(), rl2.max())
        checked += len(rows)
    assert checked >= sum(-(-len(x[3]) // 128) for x in log)
    w_gpu = st["tok_w"].cpu().numpy()
    ref_h = nx.combine(h_before, w_gpu, pool[:, :P.K], pool[:, P.K:] if P.S else None, "bf16")
    h_new = to_np(st["h"])
    assert np.array_equal(h_new, ref_h)
    assert ulp_err(to_np(st["x"]), nx.rmsnorm(h_new), "bf16") <= 1.0
    assert int(st["stats"][1]) == P.T                          # L = 1: every token retired


@pytest.mark.parametrize("d,ff,T,S", [(256, 512, 700, 0), (2048, 1408, 2048, 2), (4096, 1024, 1500, 0)])
def test_dynamic_schedules_equal_static(d, ff, T, S):
    """The dynamic tile schedules of the CTA-pair kernels (units claimed from an atomic counter —
    one list, or per-die N-tile shares with stealing — and published through a shared-memory
    ring) compute every tile with the same arithmetic as the static raster: bit-identical
    outputs, every token merged once. AMOE_FFN_SCHED is read per launch."""
    import os
    outs = []
    old = os.environ.get("AMOE_FFN_SCHED")
    try:
        for mode in ("die", "static", "dynamic", "auto"):
            os.environ["AMOE_FFN_SCHED"] = mode
            P = Problem(L=2, E=8, K=2, S=S, d=d, ff=ff, T=T, seed=23)
            ctx = P.make_ctx()
            slots = torch.arange(T, dtype=torch.int32, device="cuda")
            ctx.token_init(slots, dev_tensor(P.h0[0], "bf16"), 0)
            ctx.enqueue(0, slots, logits=torch.from_numpy(np.ascontiguousarray(P.tables[0][0, 0])).cuda())
            st = ctx.run(retire_pass=1)
            torch.cuda.synchronize()
            ctx.check()
            assert st["token_layers"] == T * 2
            outs.append(to_np(ctx.state()["h"]))
            ctx.close()
    finally:
        if old is None:
            os.environ.pop("AMOE_FFN_SCHED", None)
        else:
            os.environ["AMOE_FFN_SCHED"] = old
    assert all(np.array_equal(outs[0], o) for o in outs[1:])
