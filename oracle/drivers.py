"""Oracle drivers: synchronous fixed-batch passes and asynchronous µ-queue execution
(test infrastructure only; see oracle/__init__.py).

The paper's claim is that asynchronous layer-wise execution keeps
"the semantics of the Top-K gating function" (L153) while reordering when legs run (L189).
Both drivers call the same per-row functions in numerics.py, so their results must agree
bit-for-bit for ANY legal schedule (tested in tests/test_oracle_async.py).

Layers and passes (reading c7/c6): a token's hidden state h enters layer l as x = rmsnorm(h);
after the merge h <- h + Σ w_k O_k it moves to layer l+1; after layer L-1 it re-enters layer 0
with pass+1 (decode re-entry, PAPER.md L234 with the sampler omitted) until it retires.
"""
from __future__ import annotations

import random

import numpy as np

from . import numerics as nx
from . import scheduler as sch
from .queues import Box


def sync_run(h0, logits_fn, weights, K, n_passes=1, shared=None, dtype="bf16", record=False, gates=None):
    """Fixed-batch EP semantics: every token through layer l, then l+1.

    h0 [N, d] storage values (fp32 array); logits_fn(pass, l) -> [N, E] fp32;
    weights[l][e] = (w1, w3, w2); shared[l][j] likewise or None; gates[l] = (wg [E, d], bias
    [E] or None) routes layer l with the gate on x_l = rmsnorm(h) instead of logits_fn.
    Returns final h and (if record) the per-(pass, layer) dicts of numerics.moe_layer."""
    h = np.asarray(h0, dtype=np.float32)
    L = len(weights)
    recs = []
    for p in range(n_passes):
        for l in range(L):
            if gates is not None and gates[l] is not None:
                z = nx.gate_logits(nx.rmsnorm(h, dtype), *gates[l])
            else:
                z = logits_fn(p, l)
            r = nx.moe_layer(h, z, weights[l], K,
                             shared[l] if shared else (), dtype)
            if record:
                recs.append(r)
            h = r["h_new"]
    return h, recs


def async_run(h0, logits_fn, weights, K, G, T, n_passes=1, shared=None, dtype="bf16",
              policy="defrag", W=4, delta=0.5, max_cap=0, seed=0, combine_eagerness=0.5,
              owner=None, fault_drop=None):
    """Randomised asynchronous execution over G simulated GPUs (§3.2, §3.4).

    Each iteration either (a) picks a GPU with queued legs, selects a queue with `policy`
    (Algorithm 1 / MTFS / FLFS / random), drains up to a random cap (or all), executes the
    expert and forwards every output row to its token's pool, or (b) merges a random subset of
    tokens whose K (+S) legs all arrived, moving them to the next layer (or retiring them).
    Token id t lives on home rank t // T.  `fault_drop=(token, layer, pass, k)` silently drops
    that leg after execution (fault injection; the audit must then name the token).
    Returns (final h, box, n_token_layers)."""
    rnd = random.Random(seed)
    h = np.asarray(h0, dtype=np.float32).copy()
    N = h.shape[0]
    assert N == G * T
    L = len(weights)
    E = len(weights[0])
    S = len(shared[0]) if shared else 0
    box = Box(L, E, K, S, G, T, owner)
    layer = np.zeros(N, dtype=np.int64)
    pss = np.zeros(N, dtype=np.int64)
    x = np.zeros_like(h)
    wts = np.zeros((N, K), dtype=np.float32)
    ready = []
    done = 0
    retired = 0

    def admit(tokens):
        tokens = sorted(tokens)
        by_lp = {}
        for t in tokens:
            by_lp.setdefault((int(pss[t]), int(layer[t])), []).append(t)
        for (p, l), toks in sorted(by_lp.items()):
            toks = np.array(toks)
            x[toks] = nx.rmsnorm(h[toks], dtype)
            idx, w = nx.route_topk(logits_fn(p, l)[toks], K)
            wts[toks] = w
            box.enqueue(l, p, toks, idx, w)

    admit(range(N))
    policy_fn = None if policy == "random" else sch.POLICIES[policy]
    while retired < N:
        busy = [r for r in range(G) if any(len(box.queues[k]) for k in box.queues if k[0] == r)]
        do_combine = ready and (not busy or rnd.random() < combine_eagerness)
        if do_combine:
            rnd.shuffle(ready)
            take = ready[:rnd.randint(1, len(ready))]
            ready = ready[len(take):]
            nxt = []
            for t in take:
                legs = box.pool.pop(t)
                lg = np.stack([legs[k] for k in range(K)])[None]
                sh = np.stack([legs[K + j] for j in range(S)])[None] if S else None
                h[t] = nx.combine(h[t:t + 1], wts[t:t + 1], lg, sh, dtype)[0]
                done += 1
                layer[t] += 1
                if layer[t] == L:
                    layer[t] = 0
                    pss[t] += 1
                if pss[t] == n_passes:
                    retired += 1
                else:
                    nxt.append(t)
            if nxt:
                admit(nxt)
            continue
        if not busy:
            box.audit_quiescent()          # names the stranded token (pool not empty)
            raise AssertionError("deadlock: no queued legs and no ready tokens")
        r = rnd.choice(busy)
        Q = box.depths(r)
        if policy_fn is None:
            cand = [(l, e) for l in range(L) for e in range(E + S) if Q[l][e] > 0]
            pick = rnd.choice(cand)
        elif policy == "defrag":
            pick = policy_fn(Q, W, delta)
        else:
            pick = policy_fn(Q)
        l, e = pick
        cap = 0 if max_cap <= 0 else rnd.randint(1, max_cap)
        legs = box.drain(r, l, e, cap)
        toks = np.array([g.token for g in legs])
        wl = shared[l][e - E] if e >= E else weights[l][e]
        out = nx.expert_ffn(x[toks], *wl, dtype=dtype)
        for i, g in enumerate(legs):
            if fault_drop is not None and (g.token, g.layer, g.pass_idx, g.k) == tuple(fault_drop):
                continue
            if box.pool.put(g.token, g.k, out[i]):
                ready.append(g.token)
    box.audit_quiescent()
    return h, box, done
