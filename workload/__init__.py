"""Seeded synthetic inputs shared by the oracle tests, the CUDA parity tests and bench.py.

This package holds NO arithmetic of the method (no routing top-k, no expert FFN,
no combine, no normalisation). It only draws random numbers with the shapes and
distributions of the paper's workloads (recipe in DESIGN.md, "Inputs").
"""
from .gen import (  # noqa: F401
    WorkloadSpec,
    bf16_bits_from_f32,
    f32_from_bf16_bits,
    hidden0,
    expert_weights,
    router_logits,
    zipf_probs,
    expon_probs,
    skew_probs,
    layer_perm,
    skew_epoch,
    CONFIGS,
)
