"""Seeded synthetic workload generator (inputs only; see package docstring).

Recipe:
  * hidden states h0 ~ N(0, 1), stored as bf16 (or fp32 in fp32 mode);
  * expert weights W1, W3 ~ N(0, 1/d) with shape [ff, d]; W2 ~ N(0, 1/ff) with shape [d, ff];
  * router logits z[l, t, e] = log p[r] + Gumbel(0, 1) where p_r ∝ (r+1)^-s is a Zipf law over
    expert *ranks* r and expert e = π_l(r) for a per-layer random permutation π_l. Top-K of these
    logits is exactly a draw of K distinct experts without replacement ∝ p (Gumbel-top-k), the
    "random routing based on a profiled distribution" the paper evaluates with.
    The skew shifts: π_l is re-drawn every `shift_every` layer-steps (BASELINE.json config 4,
    reading c6 in DESIGN.md): epoch = floor((pass * L + l) / shift_every).

Every array is a pure function of (seed, stream ids). Random numbers use numpy PCG64 seeded
through SeedSequence([seed, *stream]) so different tensors never share a stream.
bf16 storage uses torch's CPU cast (round-to-nearest-even), a library routine; the oracle
and the CUDA path each decode the bits themselves.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

# stream ids (second SeedSequence word) keep the tensors independent
_S_HIDDEN, _S_W1, _S_W3, _S_W2, _S_PERM, _S_GUMBEL = 11, 21, 22, 23, 31, 41


def _rng(seed: int, *stream: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([int(seed), *map(int, stream)])))


def bf16_bits_from_f32(x: np.ndarray) -> np.ndarray:
    """fp32 array -> uint16 bf16 bit patterns (torch CPU cast, RNE)."""
    t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).to(torch.bfloat16)
    return t.view(torch.int16).numpy().view(np.uint16).copy()


def f32_from_bf16_bits(b: np.ndarray) -> np.ndarray:
    """uint16 bf16 bit patterns -> exact fp32 values (torch CPU cast)."""
    t = torch.from_numpy(np.ascontiguousarray(b, dtype=np.uint16).view(np.int16)).view(torch.bfloat16)
    return t.to(torch.float32).numpy()


@dataclass(frozen=True)
class WorkloadSpec:
    """One BASELINE.json configuration."""
    name: str
    L: int
    E: int
    K: int
    S: int
    d: int
    ff: int
    T: int            # token slots in flight per rank
    G: int = 1
    zipf_s: float = 1.2
    shift_every: int = 1000


CONFIGS = {
    # BASELINE.json configs[0]
    "tiny": WorkloadSpec("tiny", L=2, E=8, K=2, S=0, d=128, ff=256, T=512),
    # BASELINE.json configs[1]
    "mixtral": WorkloadSpec("mixtral", L=32, E=8, K=2, S=0, d=4096, ff=14336, T=16384),
    # BASELINE.json configs[2] (L=28 and per-rank T are proposals)
    "deepseek": WorkloadSpec("deepseek", L=28, E=64, K=6, S=2, d=2048, ff=1408, T=16384, G=8),
}


def zipf_probs(E: int, s: float) -> np.ndarray:
    """p_r ∝ (r+1)^-s over ranks r = 0..E-1 (float64, sums to 1)."""
    p = np.arange(1, E + 1, dtype=np.float64) ** (-float(s))
    return p / p.sum()


def expon_probs(E: int, lam: float) -> np.ndarray:
    """The paper's fitted shape ("fitted ... to an exponential distribution", no λ
    given; SPEC.md L164 uses λ ≈ 0.38): p_r ∝ exp(-λ r) over ranks r = 0..E-1 (float64)."""
    p = np.exp(-float(lam) * np.arange(E, dtype=np.float64))
    return p / p.sum()


def skew_probs(E: int, skew: str = "zipf", zipf_s: float = 1.2, lam: float = 0.38) -> np.ndarray:
    """Rank probabilities of the routing skew: 'zipf' (BASELINE.json) or 'exp' (the paper's fit)."""
    if skew == "zipf":
        return zipf_probs(E, zipf_s)
    if skew == "exp":
        return expon_probs(E, lam)
    raise ValueError(f"unknown skew {skew!r}")


def skew_epoch(pass_idx: int, l: int, L: int, shift_every: int) -> int:
    """Skew epoch of layer-step (pass, l); a 'step' is one layer traversal by the wave."""
    if shift_every <= 0:
        return 0
    return (int(pass_idx) * int(L) + int(l)) // int(shift_every)


def layer_perm(seed: int, l: int, epoch: int, E: int, same_perm: bool = False) -> np.ndarray:
    """π_l: rank r -> expert id. same_perm=True uses one permutation for all layers (worst case)."""
    g = _rng(seed, _S_PERM, 0 if same_perm else l, epoch)
    return g.permutation(E).astype(np.int32)


def router_logits(seed: int, L: int, T: int, E: int, zipf_s: float = 1.2, pass_idx: int = 0,
                  shift_every: int = 1000, same_perm: bool = False, layers=None,
                  token_offset: int = 0, skew: str = "zipf", lam: float = 0.38) -> np.ndarray:
    """Synthetic router logits, float32 [len(layers), T, E] for global tokens token_offset..+T.

    z[l, t, e] = log p[π_l^-1(e)] + Gumbel(0,1). The Gumbel noise for (pass, l) is drawn for the
    whole box-wide token range so that a rank's slice equals the corresponding slice of G=1.
    """
    if layers is None:
        layers = range(L)
    p = skew_probs(E, skew, zipf_s, lam)
    out = np.empty((len(layers), T, E), dtype=np.float32)
    for i, l in enumerate(layers):
        perm = layer_perm(seed, l, skew_epoch(pass_idx, l, L, shift_every), E, same_perm)
        logp_e = np.empty(E, dtype=np.float64)
        logp_e[perm] = np.log(p)              # expert perm[r] has probability p[r]
        g = _rng(seed, _S_GUMBEL, pass_idx, l)
        u = g.random((token_offset + T, E))[token_offset:]
        gumbel = -np.log(-np.log(np.clip(u, 1e-300, 1.0)))
        out[i] = (logp_e[None, :] + gumbel).astype(np.float32)
    return out


def hidden0(seed: int, T: int, d: int, dtype: str = "bf16", token_offset: int = 0) -> np.ndarray:
    """Initial hidden state rows ~ N(0,1). bf16 -> uint16 bits, fp32 -> float32."""
    g = _rng(seed, _S_HIDDEN)
    h = g.standard_normal((token_offset + T, d), dtype=np.float32)[token_offset:]
    return bf16_bits_from_f32(h) if dtype == "bf16" else h.copy()


def expert_weights(seed: int, l: int, e: int, d: int, ff: int, dtype: str = "bf16"):
    """(W1 [ff,d], W3 [ff,d], W2 [d,ff]) for expert e of layer l (e >= E: shared experts)."""
    w1 = _rng(seed, _S_W1, l, e).standard_normal((ff, d), dtype=np.float32) * np.float32(d ** -0.5)
    w3 = _rng(seed, _S_W3, l, e).standard_normal((ff, d), dtype=np.float32) * np.float32(d ** -0.5)
    w2 = _rng(seed, _S_W2, l, e).standard_normal((d, ff), dtype=np.float32) * np.float32(ff ** -0.5)
    if dtype == "bf16":
        return bf16_bits_from_f32(w1), bf16_bits_from_f32(w3), bf16_bits_from_f32(w2)
    return w1, w3, w2
