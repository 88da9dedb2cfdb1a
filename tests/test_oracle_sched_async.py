"""Pins of oracle/scheduler.py, oracle/queues.py and oracle/drivers.py (CPU only)."""
import json
import os

import numpy as np
import pytest

from oracle import drivers, numerics as nx, scheduler as sch
from oracle.queues import Box, ConservationError
import workload as wl


# ---------------------------------------------------------------- Algorithm 1 (worked examples)

def test_alg1_hand_executed_examples(golden_dir):
    ex = json.load(open(os.path.join(golden_dir, "alg1_examples.json")))["examples"]
    for e in ex:
        sc = sch.defrag_scores(e["Q"], e["W"], e["delta"])
        got = {f"{b},{k}": s for b, row in enumerate(sc) for k, s in enumerate(row) if s is not None}
        assert got.keys() == e["scores"].keys()
        for key, v in e["scores"].items():
            assert abs(got[key] - v) < 1e-12, key
        assert sch.defrag(e["Q"], e["W"], e["delta"]) == tuple(e["pick"])
        assert sch.mtfs(e["Q"]) == tuple(e["mtfs"])


def test_alg1_properties_random_states():
    g = np.random.default_rng(0)
    for _ in range(1000):
        NB, NE, W = g.integers(1, 12), g.integers(1, 9), int(g.integers(0, 6))
        Q = (g.integers(0, 6, (NB, NE)) * (g.random((NB, NE)) < 0.4)).tolist()
        nonempty = [(b, e) for b in range(NB) for e in range(NE) if Q[b][e] > 0]
        pick = sch.defrag(Q, W, 0.5)
        if not nonempty:
            assert pick is None and sch.mtfs(Q) is None and sch.flfs(Q) is None
            continue
        assert pick in nonempty                             # never an empty queue (L285)
        assert sch.defrag(Q, 0, 0.5) == sch.mtfs(Q)         # W=0 degenerates to MTFS
        assert sch.flfs(Q) == min(nonempty)
        if len(nonempty) == 1:
            assert pick == nonempty[0]


def test_alg1_lookahead_prefers_block_before_dense_wave():
    """With a dense wave at block b+1, a sparse queue at b outranks a bigger one elsewhere
    (the defragging intent of PAPER.md L297)."""
    Q = [[0, 0], [0, 0], [3, 0], [20, 20], [0, 0]]
    assert sch.mtfs(Q) == (3, 0)
    assert sch.defrag(Q, W=1, delta=0.9) == (2, 0)


# ---------------------------------------------------------------- µ-queues

def test_queue_fifo_and_drain_cap():
    box = Box(L=1, E=2, K=1, S=0, G=1, T=8)
    box.enqueue(0, 0, [0, 1, 2, 3], [[1], [1], [0], [1]], [[1.0]] * 4)
    assert [g.token for g in box.drain(0, 0, 1, cap=2)] == [0, 1]
    assert [g.token for g in box.drain(0, 0, 1)] == [3]
    assert [g.token for g in box.drain(0, 0, 0)] == [2]
    assert box.depths(0) == [[0, 0]]


def test_counts_equal_router_histogram_and_placement():
    T, E, K, G = 64, 8, 2, 4
    z = wl.router_logits(1, 1, G * T, E)[0]
    idx, w = nx.route_topk(z, K)
    box = Box(L=1, E=E, K=K, S=0, G=G, T=T)
    box.enqueue(0, 0, range(G * T), idx, w)
    hist = np.bincount(idx.ravel(), minlength=E)
    for e in range(E):
        q = box.queues[(e % G, 0, e)]
        assert len(q) == hist[e]
        assert all(g.home == g.token // T for g in q.q)
    assert sum(len(q) for q in box.queues.values()) == G * T * K


def test_pool_merges_exactly_k_legs():
    box = Box(L=1, E=2, K=2, S=0, G=1, T=4)
    assert box.pool.put(3, 0, 1.0) is False
    assert box.pool.put(3, 1, 2.0) is True
    assert sorted(box.pool.pop(3)) == [0, 1]
    with pytest.raises(ConservationError):
        box.pool.put(1, 0, 0.0); box.pool.put(1, 0, 0.0)


# ---------------------------------------------------------------- async == sync

def _tiny_problem(seed, L=2, E=4, K=2, S=0, d=16, ff=32, N=8, dtype="bf16"):
    h0 = wl.hidden0(seed, N, d, dtype)
    h0 = wl.f32_from_bf16_bits(h0) if dtype == "bf16" else h0
    tables = {}

    def logits(p, l):
        if (p, l) not in tables:
            tables[(p, l)] = wl.router_logits(seed, L, N, E, pass_idx=p, layers=[l])[0]
        return tables[(p, l)]

    conv = wl.f32_from_bf16_bits if dtype == "bf16" else (lambda a: a)
    W = [[tuple(conv(a) for a in wl.expert_weights(seed, l, e, d, ff, dtype)) for e in range(E)]
         for l in range(L)]
    SH = [[tuple(conv(a) for a in wl.expert_weights(seed, l, E + j, d, ff, dtype)) for j in range(S)]
          for l in range(L)] if S else None
    return h0, logits, W, SH


@pytest.mark.parametrize("G,policy,cap,S,dtype", [
    (1, "defrag", 0, 0, "bf16"), (1, "mtfs", 3, 0, "bf16"), (2, "flfs", 0, 1, "bf16"),
    (2, "random", 2, 0, "bf16"), (4, "defrag", 5, 0, "bf16"), (4, "random", 0, 1, "fp32"),
])
def test_async_equals_sync_bitwise(G, policy, cap, S, dtype):
    T = 4
    h0, logits, W, SH = _tiny_problem(G * 10 + cap, S=S, N=G * T, dtype=dtype)
    ref, _ = drivers.sync_run(h0, logits, W, K=2, n_passes=2, shared=SH, dtype=dtype)
    for seed in range(3):
        got, box, n = drivers.async_run(h0, logits, W, K=2, G=G, T=T, n_passes=2, shared=SH,
                                        dtype=dtype, policy=policy, max_cap=cap, seed=seed)
        assert n == G * T * 2 * 2
        assert np.array_equal(got, ref)


def test_async_fault_injection_names_the_token():
    h0, logits, W, _ = _tiny_problem(3, N=8)
    with pytest.raises(ConservationError, match="token 5"):
        drivers.async_run(h0, logits, W, K=2, G=2, T=4, n_passes=1, seed=1,
                          fault_drop=(5, 1, 0, 1))


def test_async_every_leg_drained_once():
    h0, logits, W, _ = _tiny_problem(4, N=8, L=3)
    _, box, _ = drivers.async_run(h0, logits, W, K=2, G=2, T=4, n_passes=2, seed=2, max_cap=2)
    drained = [(g.token, g.layer, g.pass_idx, g.k) for (_, _, _, legs) in box.trace_drain for g in legs]
    assert len(drained) == len(set(drained)) == 8 * 3 * 2 * 2


def _every_schedule(h0, logits, W, K, L, cap_choices):
    """Depth-first over every execution order of the µ-queue model on one GPU: at each step any
    nonempty (layer, expert) queue may be drained, with any cap in cap_choices (0 = drain all);
    a token merges as soon as its K legs are home (merge timing cannot change a per-token
    result). Yields the final h of every complete schedule."""
    E = len(W[0])
    N = h0.shape[0]

    def admit(st, toks, l):
        toks = np.array(sorted(toks))
        st["x"][toks] = nx.rmsnorm(st["h"][toks])
        idx, w = nx.route_topk(logits(0, l)[toks], K)
        st["w"][toks] = w
        for i, t in enumerate(toks):
            for k in range(K):
                st["q"][(l, int(idx[i, k]))].append((int(t), k))

    st0 = {"h": np.asarray(h0, np.float32).copy(), "x": np.zeros_like(h0, dtype=np.float32),
           "w": np.zeros((N, K), np.float32), "layer": [0] * N, "pool": {},
           "q": {(l, e): [] for l in range(L) for e in range(E)}, "left": N}
    admit(st0, range(N), 0)

    def step(st):
        if st["left"] == 0:
            yield st["h"]
            return
        for (l, e), q in sorted(st["q"].items()):
            if not q:
                continue
            for cap in cap_choices:
                if cap and cap >= len(q):
                    continue                        # the same as draining all
                n = len(q) if cap == 0 else cap
                s2 = {"h": st["h"].copy(), "x": st["x"], "w": st["w"].copy(), "layer": list(st["layer"]),
                      "pool": {t: dict(v) for t, v in st["pool"].items()},
                      "q": {kk: list(v) for kk, v in st["q"].items()}, "left": st["left"]}
                s2["x"] = st["x"].copy()
                legs = s2["q"][(l, e)][:n]
                s2["q"][(l, e)] = s2["q"][(l, e)][n:]
                toks = np.array([t for t, _ in legs])
                out = nx.expert_ffn(s2["x"][toks], *W[l][e])
                done = []
                for (t, k), row in zip(legs, out):
                    s2["pool"].setdefault(t, {})[k] = row
                    if len(s2["pool"][t]) == K:
                        done.append(t)
                nxt = []
                for t in done:
                    lg = s2["pool"].pop(t)
                    s2["h"][t] = nx.combine(s2["h"][t:t + 1], s2["w"][t:t + 1],
                                            np.stack([lg[k] for k in range(K)])[None])[0]
                    s2["layer"][t] += 1
                    if s2["layer"][t] == L:
                        s2["left"] -= 1
                    else:
                        nxt.append(t)
                for lyr in sorted({s2["layer"][t] for t in nxt}):
                    admit(s2, [t for t in nxt if s2["layer"][t] == lyr], lyr)
                yield from step(s2)

    yield from step(st0)


@pytest.mark.parametrize("T,E,caps,expect", [(3, 3, (0,), 12), (4, 4, (0,), 380), (3, 2, (0, 1), 38780)])
def test_async_equals_sync_over_every_schedule(T, E, caps, expect):
    """Brute force (SURVEY.md §8(c) pins): every drain order (and, in the second case, every
    drain cap) of a tiny 2-layer top-2 problem gives the synchronous result bit for bit."""
    h0, logits, W, _ = _tiny_problem(100 + T * E, N=T, E=E)
    ref, _ = drivers.sync_run(h0, logits, W, K=2, n_passes=1)
    n = 0
    for h in _every_schedule(h0, logits, W, K=2, L=2, cap_choices=caps):
        assert np.array_equal(h, ref)
        n += 1
    assert n == expect, n          # schedules enumerated for this seeded routing


def _trace_as_log(box, G):
    """The oracle async driver's own drain trace in Context.read_exec_log's format (local queue
    index := expert id, ring positions contiguous per queue)."""
    logs = [[] for _ in range(G)]
    pos = {}
    for (r, l, e, legs) in box.trace_drain:
        start = pos.get((r, l, e), 0)
        pos[(r, l, e)] = start + len(legs)
        logs[r].append((l, e, start, [(g.token % box.T, g.k, g.home, g.w, g.pass_idx) for g in legs]))
    return logs


def test_replay_accepts_a_legal_schedule_and_rejects_tampering():
    """The schedule-replay checker the GPU tests use (tests/parity_util.replay_exec_log, built on
    oracle.queues.Box.drain_given), pinned on the oracle's own randomised schedules: a legal
    drain sequence replays; a leg drained twice, a leg taken from the wrong expert's queue, a
    lost leg and a gap in a ring each fail with the token named."""
    from parity_util import replay_exec_log
    G, T, L, E, K = 2, 4, 2, 4, 2
    h0, logits, W, _ = _tiny_problem(5, N=G * T, L=L, E=E)
    _, box, _ = drivers.async_run(h0, logits, W, K=K, G=G, T=T, n_passes=2, seed=3, max_cap=2)
    logs = _trace_as_log(box, G)
    q2e = [{e: e for e in range(E)} for _ in range(G)]
    _, counts = replay_exec_log(L, E, K, 0, G, T, logits, 2, logs, q2e)
    for p in range(2):
        for l in range(L):
            idx, _ = nx.route_topk(logits(p, l), K)
            hist = np.bincount(idx.ravel(), minlength=E)
            for e in range(E):
                assert counts.get((e % G, l, e, p), 0) == hist[e]
    import copy
    dup = copy.deepcopy(logs)
    dup[0].append((dup[0][0][0], dup[0][0][1], 10 ** 6, dup[0][0][3][:1]))
    with pytest.raises((ConservationError, AssertionError)):
        replay_exec_log(L, E, K, 0, G, T, logits, 2, dup, q2e, fresh=False)
    wrong = copy.deepcopy(logs)
    l0, e0, s0, legs0 = wrong[0][0]
    wrong[0][0] = (l0, (e0 + 2) % E, s0, legs0)          # same rank, another expert's queue
    with pytest.raises((ConservationError, AssertionError)):
        replay_exec_log(L, E, K, 0, G, T, logits, 2, wrong, q2e, fresh=False)
    lost = copy.deepcopy(logs)
    l0, e0, s0, legs0 = lost[1][-1]
    lost[1][-1] = (l0, e0, s0, legs0[1:]) if len(legs0) > 1 else lost[1][-1]
    if len(legs0) > 1:
        with pytest.raises(ConservationError, match=f"token {legs0[0][2] * T + legs0[0][0]}"):
            replay_exec_log(L, E, K, 0, G, T, logits, 2, lost, q2e, fresh=False)
    gap = copy.deepcopy(logs)
    for i, (l, e, s, legs) in enumerate(gap[0]):
        if s > 0:
            gap[0][i] = (l, e, s + 1, legs)
            break
    with pytest.raises(AssertionError, match="expected"):
        replay_exec_log(L, E, K, 0, G, T, logits, 2, gap, q2e)
