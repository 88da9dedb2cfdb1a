"""Pins of oracle/numerics.py against things other than itself (CPU only)."""
import itertools
import json
import math
import os

import numpy as np
import torch

from oracle import numerics as nx
import workload as wl


# ---------------------------------------------------------------- bf16 storage (library cross-check)

def test_bf16_encode_matches_torch_cast():
    g = np.random.default_rng(0)
    x = np.concatenate([
        g.standard_normal(20000).astype(np.float32) * 10.0 ** g.integers(-30, 30, 20000),
        np.array([0.0, -0.0, np.inf, -np.inf, 1e-40, -3e-39, 65504.0, 3.3895314e38], np.float32),
        # exact ties between two bf16 values (low 16 bits = 0x8000)
        (np.arange(1000, dtype=np.uint32) << 16 | 0x8000).view(np.float32),
    ]).astype(np.float32)
    ref = torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(nx.bf16_encode(x), ref)
    assert np.array_equal(nx.bf16_decode(ref), wl.f32_from_bf16_bits(ref))


def test_bf16_nan_stays_nan():
    assert np.isnan(nx.bf16_round(np.array([np.nan], np.float32)))[0]


# ---------------------------------------------------------------- RMSNorm (closed forms)

def test_rmsnorm_constant_row_maps_to_sign():
    h = np.array([[3.0] * 64, [-0.5] * 64, [1024.0] * 64], np.float32)
    x = nx.rmsnorm(h)
    assert np.array_equal(x, np.sign(h))


def test_rmsnorm_rows_independent_and_unit_rms():
    g = np.random.default_rng(1)
    h = g.standard_normal((16, 256)).astype(np.float32) * (2.0 ** np.arange(16))[:, None]
    x = nx.rmsnorm(h, "fp32")
    rms = np.sqrt(np.mean(x.astype(np.float64) ** 2, axis=1))
    assert np.allclose(rms, 1.0, atol=1e-6)
    for i in range(16):
        assert np.array_equal(x[i], nx.rmsnorm(h[i:i + 1], "fp32")[0])
    xb = nx.rmsnorm(h, "bf16")
    assert np.allclose(np.sqrt(np.mean(xb.astype(np.float64) ** 2, axis=1)), 1.0, atol=4e-3)


# ---------------------------------------------------------------- router (brute force + library)

def test_route_topk_brute_force_subsets():
    g = np.random.default_rng(2)
    E, K = 6, 3
    z = g.standard_normal((200, E)).astype(np.float32)
    idx, w = nx.route_topk(z, K)
    for t in range(200):
        # unique max-sum K-subset for distinct logits
        best = max(itertools.combinations(range(E), K), key=lambda s: sum(float(z[t, e]) for e in s))
        assert set(idx[t]) == set(best)
        assert all(z[t, idx[t, k]] >= z[t, idx[t, k + 1]] for k in range(K - 1))
    # softmax over the selected logits (library routine, float64)
    sel = torch.from_numpy(np.take_along_axis(z, idx, 1).astype(np.float64))
    assert np.allclose(w, torch.softmax(sel, dim=1).numpy(), rtol=0, atol=1e-7)
    assert np.allclose(w.sum(1), 1.0, atol=1e-6)


def test_route_topk_ties_go_to_lower_index():
    z = np.array([[1.0, 3.0, 3.0, 0.0, 3.0]], np.float32)
    idx, w = nx.route_topk(z, 2)
    assert idx.tolist() == [[1, 2]]
    assert np.allclose(w, [[0.5, 0.5]])
    idx, _ = nx.route_topk(np.zeros((1, 4), np.float32), 3)
    assert idx.tolist() == [[0, 1, 2]]


def test_route_topk_matches_torch_topk_on_distinct_logits():
    g = np.random.default_rng(3)
    z = g.standard_normal((500, 64)).astype(np.float32)
    idx, _ = nx.route_topk(z, 6)
    ref = torch.topk(torch.from_numpy(z), 6, dim=1).indices.numpy()
    assert np.array_equal(idx, ref)


def _exact_inclusion(p, K):
    """P(expert i among K draws without replacement ∝ p), by exhaustive recursion."""
    E = len(p)
    incl = np.zeros(E)

    def rec(chosen, prob, left):
        if len(chosen) == K:
            for e in chosen:
                incl[e] += prob
            return
        for e in range(E):
            if e not in chosen:
                rec(chosen + [e], prob * p[e] / left, left - p[e])
    rec([], 1.0, 1.0)
    return incl


def test_gumbel_topk_is_sampling_without_replacement():
    """Zipf s=1.2, E=8, K=2: Gumbel-top-k of the generator's logits through the oracle router
    reproduces exact sequential sampling without replacement (SURVEY.md §8(c) router pin)."""
    E, K, T = 8, 2, 40000
    p = wl.zipf_probs(E, 1.2)
    exact = _exact_inclusion(p, K)
    assert np.allclose(exact[:3], [0.7055, 0.4043, 0.2600], atol=1e-4)
    z = wl.router_logits(seed=5, L=1, T=T, E=E, same_perm=True)[0]
    perm = wl.layer_perm(5, 0, 0, E, same_perm=True)
    idx, _ = nx.route_topk(z, K)
    cnt = np.bincount(idx.ravel(), minlength=E) / T
    mc = cnt[perm]                                   # frequency of rank r
    se = np.sqrt(exact * (1 - exact) / T)
    assert np.all(np.abs(mc - exact) < 4 * se + 1e-9)
    assert abs(mc[0] / K - 0.3527) < 0.01            # hottest expert's share of legs


# ---------------------------------------------------------------- SwiGLU expert

def _brute_ffn(x, w1, w3, w2, dtype):
    """Pure-Python scalar loops (independent of BLAS): the definition on tiny inputs."""
    n, d = x.shape
    ff = w1.shape[0]
    out = np.zeros((n, w2.shape[0]), np.float32)
    for i in range(n):
        a = []
        for j in range(ff):
            gsum = math.fsum(float(x[i, c]) * float(w1[j, c]) for c in range(d))
            usum = math.fsum(float(x[i, c]) * float(w3[j, c]) for c in range(d))
            gv, uv = float(np.float32(gsum)), float(np.float32(usum))
            a.append(gv / (1.0 + math.exp(-gv)) * uv)
        a = nx.to_storage(np.array(a), dtype)
        for o in range(w2.shape[0]):
            out[i, o] = np.float32(math.fsum(float(a[j]) * float(w2[o, j]) for j in range(ff)))
    return nx.to_storage(out, dtype)


def test_expert_ffn_equals_brute_force_loops():
    g = np.random.default_rng(4)
    n, d, ff = 3, 4, 5                                    # d != ff catches transposed operands
    for dtype in ("bf16", "fp32"):
        x = nx.to_storage(g.standard_normal((n, d)), dtype)
        w1 = nx.to_storage(g.standard_normal((ff, d)) * 0.5, dtype)
        w3 = nx.to_storage(g.standard_normal((ff, d)) * 0.5, dtype)
        w2 = nx.to_storage(g.standard_normal((d, ff)) * 0.5, dtype)
        got = nx.expert_ffn(x, w1, w3, w2, dtype)
        ref = _brute_ffn(x, w1, w3, w2, dtype)
        # float64 BLAS vs exact fsum can differ only in the last fp32 ulp before rounding
        assert np.allclose(got, ref, rtol=1e-6 if dtype == "fp32" else 8e-3, atol=0)


def test_expert_ffn_textbook_silu_values(golden_dir):
    """One-hot weights route known gate values g and up values u to known outputs:
    O[i, o] = silu(g_i) * u_i exactly (rounded). Gate/up swapped or W2 transposed fails."""
    table = json.load(open(os.path.join(golden_dir, "swiglu_textbook.json")))["silu"]
    gs = np.array([float(k) for k in table], np.float32)
    n = len(gs)
    d, ff = 3, 4
    x = np.zeros((n, d), np.float32)
    x[:, 0] = gs                                         # feature 0 carries g
    x[:, 1] = 1.0                                        # feature 1 is a constant 1
    w1 = np.zeros((ff, d), np.float32); w1[2, 0] = 1.0  # gate unit 2 reads g
    w3 = np.zeros((ff, d), np.float32); w3[2, 1] = 3.0  # up unit 2 = 3
    w2 = np.zeros((d, ff), np.float32); w2[1, 2] = 1.0  # output feature 1 = activation 2
    got = nx.expert_ffn(x, w1, w3, w2, "fp32")
    want = np.array([3.0 * v for v in table.values()], np.float32)
    assert np.allclose(got[:, 1], want, rtol=1e-7, atol=1e-7)
    assert np.all(got[:, 0] == 0) and np.all(got[:, 2] == 0)


def test_expert_ffn_row_independent_bitwise():
    """Batch invariance: a row's output does not depend on its batch (n = 1..64)."""
    g = np.random.default_rng(6)
    d, ff = 64, 96
    x = nx.bf16_round(g.standard_normal((64, d)))
    w1, w3, w2 = (nx.bf16_round(g.standard_normal(s) / np.sqrt(s[1])) for s in ((ff, d), (ff, d), (d, ff)))
    full = nx.expert_ffn(x, w1, w3, w2)
    for n in (1, 2, 7, 33):
        assert np.array_equal(nx.expert_ffn(x[:n], w1, w3, w2), full[:n])
    assert np.array_equal(nx.expert_ffn(x[40:41], w1, w3, w2)[0], full[40])


def test_single_expert_top1_is_dense_swiglu_mlp():
    """E=1, K=1: the MoE layer is h + SwiGLU(rmsnorm(h)) (special case of the method)."""
    g = np.random.default_rng(7)
    T, d, ff = 10, 32, 48
    h = nx.bf16_round(g.standard_normal((T, d)))
    W = [tuple(nx.bf16_round(g.standard_normal(s) / np.sqrt(s[1])) for s in ((ff, d), (ff, d), (d, ff)))]
    r = nx.moe_layer(h, np.zeros((T, 1), np.float32), W, K=1)
    assert np.all(r["idx"] == 0) and np.all(r["w"] == 1.0)
    x = nx.rmsnorm(h)
    assert np.array_equal(r["h_new"], nx.bf16_round(h + nx.expert_ffn(x, *W[0])))


# ---------------------------------------------------------------- combine (closed forms)

def test_combine_exact_examples():
    h = np.array([[1.0, -2.0]], np.float32)
    w = np.array([[0.75, 0.25]], np.float32)
    legs = np.array([[[4.0, 8.0], [8.0, -16.0]]], np.float32)
    assert nx.combine(h, w, legs).tolist() == [[1 + 3 + 2, -2 + 6 - 4]]
    # one-hot weights select a single leg
    w1h = np.array([[0.0, 1.0]], np.float32)
    assert nx.combine(h, w1h, legs, dtype="fp32").tolist() == [[9.0, -18.0]]
    # shared experts enter with weight 1 after the routed legs
    sh = np.array([[[0.5, 0.5]]], np.float32)
    assert nx.combine(h, w, legs, sh, dtype="fp32").tolist() == [[6.5, 0.5]]


def test_combine_order_is_ascending_k():
    """fp32 addition is not associative: the merge order is fixed (reading c9).
    1 + 2^-24 + 2^-24 in that order gives 1, but (2^-24 + 2^-24) + 1 would give 1 + 2^-23."""
    eps = np.float32(2.0 ** -24)
    h = np.array([[1.0]], np.float32)
    legs = np.array([[[eps], [eps]]], np.float32)
    out = nx.combine(h, np.ones((1, 2), np.float32), legs, dtype="fp32")
    assert out[0, 0] == np.float32(1.0)


def test_combine_constant_legs_return_the_leg():
    g = np.random.default_rng(8)
    w = g.random((50, 4)).astype(np.float32)
    w /= w.sum(1, keepdims=True)
    o = nx.bf16_round(g.standard_normal((50, 1, 16)))
    legs = np.repeat(o, 4, axis=1)
    out = nx.combine(np.zeros((50, 16), np.float32), w, legs)
    assert np.allclose(out, o[:, 0], rtol=8e-3, atol=0)


def test_gate_logits_brute_force_and_one_hot():
    """Router gate (f3): z = x·Wgᵀ + b. Pinned by pure-Python fsum loops on a tiny shape, by
    one-hot gate rows (z_e = x_{j(e)} exactly) and by the bias alone (Wg = 0 -> z = b)."""
    import math
    rng = np.random.default_rng(3)
    x = rng.standard_normal((5, 7)).astype(np.float32)
    wg = rng.standard_normal((4, 7)).astype(np.float32)
    b = rng.standard_normal(4).astype(np.float32)
    z = nx.gate_logits(x, wg, b)
    for t in range(5):
        for e in range(4):
            ref = math.fsum(float(x[t, j]) * float(wg[e, j]) for j in range(7)) + float(b[e])
            assert abs(float(z[t, e]) - ref) <= 1e-6 * max(1.0, abs(ref))
    onehot = np.zeros((4, 7), np.float32)
    cols = [6, 0, 3, 3]
    for e, j in enumerate(cols):
        onehot[e, j] = 1.0
    assert np.array_equal(nx.gate_logits(x, onehot), x[:, cols])
    assert np.array_equal(nx.gate_logits(x, np.zeros((4, 7), np.float32), b), np.tile(b, (5, 1)))
    # routing with a one-hot gate picks the largest coordinates of x among `cols`
    idx, _ = nx.route_topk(nx.gate_logits(x, onehot), 1)
    assert all(x[t, cols[idx[t, 0]]] == max(x[t, c] for c in cols) for t in range(5))


# ---------------------------------------------------------------- SURVEY.md §8(c) FFN pins


def _experts(g, E, d, ff):
    return [tuple(nx.bf16_round(g.standard_normal(s) / np.sqrt(s[1])) for s in ((ff, d), (ff, d), (d, ff)))
            for _ in range(E)]


def test_k_equals_e_with_equal_logits_is_the_mean_of_the_experts():
    """K = E with equal logits: every token visits every expert in index order (tie rule c12)
    with weight exactly 1/E (softmax of equal values, E a power of two), so the layer adds the
    plain mean of all experts' outputs — the closed form, evaluated in float64 here, must agree
    within the storage rounding of h_new (one bf16 ulp) on every element. A dropped leg, a
    wrong weight or a leg merged twice moves rows by ~1/E of an expert output."""
    g = np.random.default_rng(21)
    T, E, d, ff = 12, 4, 32, 48
    h = nx.bf16_round(g.standard_normal((T, d)))
    W = _experts(g, E, d, ff)
    r = nx.moe_layer(h, np.zeros((T, E), np.float32), W, K=E)
    assert np.array_equal(r["idx"], np.tile(np.arange(E), (T, 1)))
    assert np.all(r["w"] == np.float32(1.0 / E))
    x = nx.rmsnorm(h)
    mean = np.mean([nx.expert_ffn(x, *w).astype(np.float64) for w in W], axis=0)
    ref = h.astype(np.float64) + mean
    ulp = 2.0 ** (np.floor(np.log2(np.maximum(np.abs(ref), 1e-30))) - 7)
    assert np.all(np.abs(r["h_new"] - ref) <= ulp)
    # a layer with one expert's leg dropped is far outside that bound
    legs = r["legs"].copy()
    legs[:, E - 1] = 0
    bad = nx.combine(h, r["w"], legs)
    assert np.max(np.abs(bad - ref) / ulp) > 4


def test_point_mass_router_uses_only_expert_zero():
    """A router whose logits put all mass on expert 0 (others -inf) with K = 1: every token's
    single leg goes to expert 0 with weight 1, so the layer is h + SwiGLU_0(rmsnorm(h)) and the
    other experts' weights are never read (replacing them with NaN changes nothing)."""
    g = np.random.default_rng(22)
    T, E, d, ff = 9, 8, 32, 64
    h = nx.bf16_round(g.standard_normal((T, d)))
    W = _experts(g, E, d, ff)
    z = np.full((T, E), -np.inf, np.float32)
    z[:, 0] = 0.0
    r = nx.moe_layer(h, z, W, K=1)
    assert np.all(r["idx"] == 0) and np.all(r["w"] == 1.0)
    x = nx.rmsnorm(h)
    assert np.array_equal(r["h_new"], nx.bf16_round(h + nx.expert_ffn(x, *W[0])))
    Wn = [W[0]] + [tuple(np.full_like(a, np.nan) for a in w) for w in W[1:]]
    assert np.array_equal(nx.moe_layer(h, z, Wn, K=1)["h_new"], r["h_new"])
