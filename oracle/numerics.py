"""Oracle arithmetic of one MoE layer (test infrastructure only; see oracle/__init__.py).

Rounding points (reading c8): values are stored in bf16 (or fp32 in fp32 mode),
GEMMs accumulate in float64 and are rounded to fp32 (the GPU accumulates in fp32 TMEM), the
SwiGLU activation is rounded to the storage type, the down projection is rounded to fp32 then
to storage, the combine accumulates in fp32 with separate multiply and add (no FMA).
"""
from __future__ import annotations

import numpy as np

# ----------------------------------------------------------------------------- storage types


def bf16_decode(bits: np.ndarray) -> np.ndarray:
    """uint16 bf16 bit patterns -> fp32 values (the bf16 value is the top half of an fp32)."""
    return (np.asarray(bits, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


def bf16_encode(x: np.ndarray) -> np.ndarray:
    """float -> uint16 bf16 bits, round-to-nearest-even on the fp32 bit pattern.

    float64 input is first rounded to fp32 (the GPU's last arithmetic is fp32)."""
    u = np.ascontiguousarray(np.asarray(x, dtype=np.float32)).view(np.uint32).astype(np.uint64)
    nan = (u & 0x7FFFFFFF) > 0x7F800000
    r = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
    r = np.where(nan, (u >> 16) | 0x40, r)
    return (r & 0xFFFF).astype(np.uint16)


def bf16_round(x: np.ndarray) -> np.ndarray:
    """float -> nearest bf16 value, returned as fp32."""
    return bf16_decode(bf16_encode(x))


def to_storage(x: np.ndarray, dtype: str) -> np.ndarray:
    """Round to the storage type, returned as fp32 values."""
    return bf16_round(x) if dtype == "bf16" else np.asarray(x, dtype=np.float32)


# ----------------------------------------------------------------------------- c7: RMSNorm

RMS_EPS = 1e-6


def rmsnorm(h: np.ndarray, dtype: str = "bf16", eps: float = RMS_EPS) -> np.ndarray:
    """x = h / sqrt(mean(h^2) + eps), per row, rounded to storage (reading c7).

    The paper puts attention + gating between expert layers ("We consider MoE's
    gating and top-K merge operators as part of the attention layer"); attention is out of
    scope, and a weightless pre-norm keeps random-weight chains finite."""
    h64 = np.asarray(h, dtype=np.float64)
    ms = np.mean(h64 * h64, axis=-1, keepdims=True)
    return to_storage(h64 / np.sqrt(ms + eps), dtype)


# ----------------------------------------------------------------------------- a1: router


def route_topk(z: np.ndarray, K: int):
    """Router top-k ("After routing ... a token is duplicated K times and
    dispatched to K different experts"; L202 "Topk_weights: used for top-k token merging").

    idx[t] = the K largest logits in descending order, ties -> lower expert index (reading c12);
    w[t,k] = softmax over the K selected logits (reading c2), in float64, rounded to fp32.
    """
    z = np.asarray(z, dtype=np.float32)
    T, E = z.shape
    idx = np.empty((T, K), dtype=np.int32)
    w = np.empty((T, K), dtype=np.float32)
    for t in range(T):
        order = sorted(range(E), key=lambda e: (-float(z[t, e]), e))[:K]
        idx[t] = order
        sel = z[t, order].astype(np.float64)
        ex = np.exp(sel - sel[0])
        w[t] = (ex / ex.sum()).astype(np.float32)
    return idx, w


def gate_logits(x: np.ndarray, wg: np.ndarray, bias: np.ndarray | None = None) -> np.ndarray:
    """Router gate ("gating" is the last op of the attention layer, PAPER.md
    L175): z[t, e] = Σ_j x[t, j]·wg[e, j] + bias[e], accumulated in float64, rounded to fp32."""
    z = np.asarray(x, np.float64) @ np.asarray(wg, np.float64).T
    if bias is not None:
        z = z + np.asarray(bias, np.float64)[None, :]
    return z.astype(np.float32)


# ----------------------------------------------------------------------------- a5-a6: expert


def silu(g: np.ndarray) -> np.ndarray:
    """silu(g) = g / (1 + e^-g) (SwiGLU gate activation, reading c1)."""
    g = np.asarray(g, dtype=np.float64)
    return g / (1.0 + np.exp(-g))


def expert_ffn(x: np.ndarray, w1: np.ndarray, w3: np.ndarray, w2: np.ndarray,
               dtype: str = "bf16") -> np.ndarray:
    """One expert over a drained batch: O = W2 · (silu(W1·x) ⊙ W3·x) per row (reading c1).

    x [n, d], w1/w3 [ff, d], w2 [d, ff] are exact storage values (fp32 arrays).
    Each output row depends only on its own input row (no cross-row arithmetic), which is what
    makes asynchronous re-batching return the synchronous result.
    """
    A = swiglu_act(x, w1, w3, dtype)
    O = (A.astype(np.float64) @ np.asarray(w2, np.float64).T).astype(np.float32)
    return to_storage(O, dtype)


def swiglu_act(x: np.ndarray, w1: np.ndarray, w3: np.ndarray, dtype: str = "bf16") -> np.ndarray:
    """The expert's hidden activation A = store(silu(fp32(W1·x)) ⊙ fp32(W3·x)), [n, ff]."""
    x64 = np.asarray(x, dtype=np.float64)
    G = (x64 @ np.asarray(w1, np.float64).T).astype(np.float32)
    U = (x64 @ np.asarray(w3, np.float64).T).astype(np.float32)
    return to_storage(silu(G) * U.astype(np.float64), dtype)


# ----------------------------------------------------------------------------- a8: combine


def combine(h: np.ndarray, w: np.ndarray, legs: np.ndarray, shared: np.ndarray | None = None,
            dtype: str = "bf16") -> np.ndarray:
    """Top-K token merge (duplicated tokens "are merged into a single token";
    L175: the merge is the first operator of the next block).

    h_new = store( fp32(h) + Σ_{k<K} w_k·O_k + Σ_{j<S} O^shared_j ), accumulated left to right
    in ascending k then j (reading c9), every multiply and add rounded to fp32 separately.
    h [T, d]; w [T, K]; legs [T, K, d]; shared [T, S, d] or None.
    """
    acc = np.asarray(h, dtype=np.float32).copy()
    w = np.asarray(w, dtype=np.float32)
    legs = np.asarray(legs, dtype=np.float32)
    for k in range(legs.shape[1]):
        prod = (w[:, k:k + 1] * legs[:, k, :]).astype(np.float32)
        acc = (acc + prod).astype(np.float32)
    if shared is not None:
        for j in range(shared.shape[1]):
            acc = (acc + np.asarray(shared[:, j, :], np.float32)).astype(np.float32)
    return to_storage(acc, dtype)


# ----------------------------------------------------------------------------- full layer


def moe_layer(h: np.ndarray, z: np.ndarray, weights, K: int, shared_weights=(), dtype="bf16"):
    """One synchronous MoE layer (fixed-batch EP semantics).

    h [T,d] storage values; z [T,E] logits; weights[e] = (w1, w3, w2); shared_weights[j] likewise.
    Returns dict(x, idx, w, legs [T,K,d], shared [T,S,d] or None, h_new)."""
    x = rmsnorm(h, dtype)
    idx, w = route_topk(z, K)
    T, d = x.shape
    legs = np.zeros((T, K, d), dtype=np.float32)
    for e in range(len(weights)):
        rows = [(t, k) for t in range(T) for k in range(K) if idx[t, k] == e]
        if not rows:
            continue
        tok = np.array([t for t, _ in rows])
        out = expert_ffn(x[tok], *weights[e], dtype=dtype)
        for i, (t, k) in enumerate(rows):
            legs[t, k] = out[i]
    sh = None
    if shared_weights:
        sh = np.stack([expert_ffn(x, *sw, dtype=dtype) for sw in shared_weights], axis=1)
    h_new = combine(h, w, legs, sh, dtype)
    return dict(x=x, idx=idx, w=w, legs=legs, shared=sh, h_new=h_new)
