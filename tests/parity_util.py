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
