"""Helpers shared by the GPU parity tests: build a libamoe context from the seeded workload,
and the tolerance metrics of DESIGN.md reading c13."""
from __future__ import annotations

import numpy as np
import torch

import workload as wl
from oracle import numerics as nx

TOL = {"bf16": 2e-2, "fp32": 1e-5}        # BASELINE.json north_star
ROW_L2 = {"bf16": 2e-3, "fp32": 1e-6}     # diagnostic gate


def floored_err(got: np.ndarray, ref: np.ndarray) -> float:
    """max |got - ref| / max(|ref|, rms(ref row)) over all elements (reading c13)."""
    got = np.asarray(got, np.float64).reshape(-1, ref.shape[-1])
    ref = np.asarray(ref, np.float64).reshape(-1, ref.shape[-1])
    rms = np.sqrt(np.mean(ref * ref, axis=1, keepdims=True)) + 1e-30
    return float(np.max(np.abs(got - ref) / np.maximum(np.abs(ref), rms))) if ref.size else 0.0


def row_l2_err(got: np.ndarray, ref: np.ndarray) -> float:
    """Mean over rows of ‖got - ref‖₂ / ‖ref‖₂ (diagnostic; a systematic bug — a wrong operand,
    truncation instead of RNE, a missing rounding — raises every row, rounding-order noise does
    not. The max over rows is shape-dependent noise at small widths, hence the mean)."""
    got = np.asarray(got, np.float64).reshape(-1, ref.shape[-1])
    ref = np.asarray(ref, np.float64).reshape(-1, ref.shape[-1])
    if not ref.size:
        return 0.0
    return float(np.mean(np.linalg.norm(got - ref, axis=1) / (np.linalg.norm(ref, axis=1) + 1e-30)))


def ulp_err(got: np.ndarray, ref: np.ndarray, dtype: str) -> float:
    """max |got - ref| in units of the storage type's ulp at |ref|."""
    ref = np.asarray(ref, np.float64)
    mant = 8 if dtype == "bf16" else 24
    ulp = 2.0 ** (np.floor(np.log2(np.maximum(np.abs(ref), 1e-30))) - (mant - 1))
    return float(np.max(np.abs(np.asarray(got, np.float64) - ref) / ulp)) if ref.size else 0.0


def to_np(t: torch.Tensor) -> np.ndarray:
    return t.detach().float().cpu().numpy()


def dev_tensor(arr: np.ndarray, dtype: str, device="cuda") -> torch.Tensor:
    """Generator output (uint16 bf16 bits or fp32) -> device tensor of the storage type."""
    if dtype == "bf16":
        return torch.from_numpy(np.ascontiguousarray(arr).view(np.int16)).view(torch.bfloat16).to(device)
    return torch.from_numpy(np.ascontiguousarray(arr, dtype=np.float32)).to(device)


def host_values(arr: np.ndarray, dtype: str) -> np.ndarray:
    return wl.f32_from_bf16_bits(arr) if dtype == "bf16" else np.asarray(arr, np.float32)


class Problem:
    """Seeded workload for one config: device weights registered in ctx(s) and oracle copies."""

    def __init__(self, L, E, K, S, d, ff, T, G=1, dtype="bf16", seed=0, n_tab=2, zipf_s=1.2):
        self.L, self.E, self.K, self.S, self.d, self.ff, self.T, self.G = L, E, K, S, d, ff, T, G
        self.dtype, self.seed, self.n_tab = dtype, seed, n_tab
        self.W = {}        # (l, e) -> oracle (w1, w3, w2) fp32 values
        self.Wd = {}       # (l, e) -> device tensors
        for l in range(L):
            for e in range(E + S):
                raw = wl.expert_weights(seed, l, e, d, ff, dtype)
                self.W[(l, e)] = tuple(host_values(a, dtype) for a in raw)
                self.Wd[(l, e)] = tuple(dev_tensor(a, dtype) for a in raw)
        # router tables per rank: [n_tab][L][T][E] over this rank's token slots
        self.tables = []
        for r in range(G):
            tab = np.stack([wl.router_logits(seed, L, T, E, zipf_s=zipf_s, pass_idx=p, token_offset=r * T)
                            for p in range(n_tab)])
            self.tables.append(tab)
        self.h0 = [wl.hidden0(seed, T, d, dtype, token_offset=r * T) for r in range(G)]

    def logits(self, p, l):
        """Box-wide [G*T, E] logits of (pass, layer) for the oracle."""
        return np.concatenate([t[p % self.n_tab, l] for t in self.tables], axis=0)

    def oracle_weights(self):
        W = [[self.W[(l, e)] for e in range(self.E)] for l in range(self.L)]
        SH = [[self.W[(l, self.E + j)] for j in range(self.S)] for l in range(self.L)] if self.S else None
        return W, SH

    def make_ctx(self, rank=0, max_batch=0, rows_cap=0, owner=None):
        from paper_2505_08944_b200 import amoe
        cfg = amoe.make_config(self.L, self.E, self.K, self.S, self.d, self.ff, self.T, G=self.G, rank=rank,
                               dtype=self.dtype, max_batch=max_batch, rows_cap=rows_cap, owner=owner)
        ctx = amoe.Context(cfg)
        for l in range(self.L):
            for e in range(self.E + self.S):
                if e >= self.E or ctx.local_queue(e) >= 0 and (owner[e] if owner else e % self.G) == rank:
                    ctx.set_expert(l, e, *self.Wd[(l, e)])
        ctx.set_router(torch.from_numpy(self.tables[rank]).cuda().contiguous())
        return ctx


def replay_exec_log(L, E, K, S, G, T, logits_fn, n_passes, logs, q2e, fresh=True):
    """Schedule replay. logs[r] = rank r's drains in order, each
    (layer, local queue, ring start, [(slot, k, home, w, pass), ...]) as Context.read_exec_log
    returns them; q2e[r] maps rank r's local queue index to the expert id (E + j = shared j).
    The oracle's µ-queue model (oracle.queues.Box over G ranks) is filled with every routed leg
    of passes 0..n_passes-1 (routing is a pure function of the synthetic logits), then every
    logged drain is replayed through Box.drain_given, which checks bit-exactly that each drained
    leg was queued at that (rank, layer, expert) for that pass and is taken once. Also checked:
    consecutive drains of a ring are contiguous (each takes the oldest entries after the last
    one, from position 0 on a fresh context), each leg's weight is the router's (|Δw| <= 1e-6),
    and at the end every leg was drained exactly once (Box.audit_quiescent names a lost one).
    Returns the Box and the per-(rank, layer, expert, pass) drained counts."""
    from oracle.queues import Box
    box = Box(L=L, E=E, K=K, S=S, G=G, T=T)
    wref = {}
    for p in range(n_passes):
        for l in range(L):
            idx, w = nx.route_topk(logits_fn(p, l), K)
            box.enqueue(l, p, range(G * T), idx, w)
            for t in range(G * T):
                for k in range(K):
                    wref[(t, k, p, l)] = float(w[t, k])
    counts = {}
    for r, log in enumerate(logs):
        nxt = {}
        for (l, q, start, legs) in log:
            e = q2e[r][q]
            if (l, q) in nxt:
                assert start == nxt[(l, q)], f"rank {r} ring ({l},{q}): drain at {start}, expected {nxt[(l, q)]}"
            elif fresh:
                assert start == 0, f"rank {r} ring ({l},{q}): first drain at {start}"
            nxt[(l, q)] = start + len(legs)
            keys = [(home * T + slot, k, ps) for slot, k, home, _, ps in legs]
            box.drain_given(r, l, e, keys)
            for (slot, k, home, wv, ps) in legs:
                ref = wref[(home * T + slot, k, ps, l)] if k < K else 1.0
                assert abs(wv - ref) <= 1e-6, (r, l, e, slot, k, wv, ref)
                key = (r, l, e, ps)
                counts[key] = counts.get(key, 0) + 1
    box.audit_quiescent()
    return box, counts
