"""The seeded input generator: determinism, rank slicing, distributions (CPU only)."""
import numpy as np

import workload as wl


def test_generator_is_deterministic_and_slices_by_rank():
    a = wl.router_logits(3, L=2, T=64, E=8)
    b = wl.router_logits(3, L=2, T=64, E=8)
    assert a.tobytes() == b.tobytes()
    s = wl.router_logits(3, L=2, T=32, E=8, token_offset=32)
    assert np.array_equal(s, a[:, 32:])
    assert np.array_equal(wl.hidden0(1, 10, 16, token_offset=6), wl.hidden0(1, 16, 16)[6:])
    w1, w3, w2 = wl.expert_weights(0, 1, 2, 32, 48)
    assert w1.shape == (48, 32) and w3.shape == (48, 32) and w2.shape == (32, 48)
    assert w1.dtype == np.uint16 and not np.array_equal(w1, w3)


def test_zipf_probs_and_skew_epochs():
    p = wl.zipf_probs(8, 1.2)
    assert abs(p.sum() - 1) < 1e-15 and np.all(np.diff(p) < 0)
    assert abs(p[0] / p[1] - 2 ** 1.2) < 1e-12
    assert wl.skew_epoch(0, 31, 32, 1000) == 0 and wl.skew_epoch(31, 8, 32, 1000) == 1
    assert not np.array_equal(wl.layer_perm(0, 0, 0, 64), wl.layer_perm(0, 0, 1, 64))
    assert np.array_equal(np.sort(wl.layer_perm(0, 5, 2, 64)), np.arange(64))


def test_weight_scales():
    w1, _, w2 = wl.expert_weights(0, 0, 0, 512, 1024, dtype="fp32")
    assert abs(w1.std() - 512 ** -0.5) < 0.01 * 512 ** -0.5 * 10
    assert abs(w2.std() - 1024 ** -0.5) < 0.01 * 1024 ** -0.5 * 10


def test_exponential_skew_variant():
    """The paper's exponential fit (λ = 0.38 from SPEC.md L164): p_r ∝ e^{-λr}."""
    p = wl.expon_probs(8, 0.38)
    assert abs(p.sum() - 1) < 1e-15
    assert np.allclose(p[:-1] / p[1:], np.exp(0.38), rtol=1e-12)
    assert np.array_equal(wl.skew_probs(8, "zipf"), wl.zipf_probs(8, 1.2))
    z = wl.router_logits(0, L=1, T=20000, E=8, skew="exp")[0]
    top1 = np.bincount(z.argmax(axis=1), minlength=8) / 20000.0
    perm = wl.layer_perm(0, 0, 0, 8)
    # argmax of log p + Gumbel is a draw from p: the top-1 share of each expert matches p
    assert np.abs(top1[perm] - p).max() < 0.015


def test_hottest_expert_share_matches_survey():
    """Zipf s = 1.2 routing (Gumbel-top-k): the hottest expert's share of all legs is ≈ 0.3524
    for E = 8, K = 2 and ≈ 0.1516 for E = 64, K = 6 (SURVEY.md §8(c) pins, Monte Carlo there);
    20000 tokens give a standard error below 0.003."""
    for E, K, share in [(8, 2, 0.3524), (64, 6, 0.1516)]:
        z = wl.router_logits(0, 1, 20000, E)[0]
        idx = np.argsort(-z, axis=1, kind="stable")[:, :K]
        got = np.bincount(idx.ravel(), minlength=E).max() / idx.size
        assert abs(got - share) < 0.006, (E, K, got)


def test_skew_shift_redraws_layer_permutations():
    """Skew shifting (BASELINE.json configs[3], reading c6): with a 32-layer wave and an epoch of
    32 layer-steps, pass 0 and pass 1 fall in different epochs, so every layer's expert
    permutation is redrawn (the hot expert moves for most layers), while passes in the same epoch
    share it. Checked on the generated logits, not only on skew_epoch."""
    L, T, E = 32, 4000, 8
    z0 = wl.router_logits(3, L, T, E, pass_idx=0, shift_every=32)
    z1 = wl.router_logits(3, L, T, E, pass_idx=1, shift_every=32)
    z0b = wl.router_logits(3, L, T, E, pass_idx=0, shift_every=1000)
    z1b = wl.router_logits(3, L, T, E, pass_idx=1, shift_every=1000)
    hot = lambda z: np.bincount(z.argmax(axis=1), minlength=E).argmax()
    moved = sum(hot(z0[l]) != hot(z1[l]) for l in range(L))
    same = sum(hot(z0b[l]) != hot(z1b[l]) for l in range(L))
    assert moved >= L // 2          # a fresh permutation per layer: the hottest expert moves (7/8 chance)
    assert same == 0                # one epoch: same permutation, only the Gumbel noise differs
