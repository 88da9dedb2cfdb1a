"""Top-1 direct forwarding (amoe_set_direct): with
K = 1 the executing rank merges, normalises, routes and scatters each token itself — no token
pool, no combine ring, no merge launch on the home.

- counts: every token-layer merged once, every leg executed once (bit-exact);
- numerics: h against the float64 oracle's synchronous top-1 run (floored 2e-2, row-L2 2e-3,
  reading c13; the 2-layer tiny config runs free);
- the pooled path (amoe_combine) on the same schedule gives the same h bit for bit (same merge
  arithmetic, no FMA), so direct forwarding changes where the merge runs, not what it computes;
- at G = 2 (loopback contexts, router gate on every layer) legs cross ranks: the executing rank
  updates the remote home's h / x / token state and counters over peer memory.
"""
import numpy as np
import pytest
import torch

from oracle import drivers
from parity_util import ROW_L2, TOL, Problem, dev_tensor, floored_err, host_values, row_l2_err, to_np

pytestmark = pytest.mark.gpu

TOP1 = dict(L=2, E=8, K=1, S=0, d=128, ff=256, T=512)


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    from paper_2505_08944_b200 import build
    build.build()


def _run(P, direct, passes=2):
    ctx = P.make_ctx()
    if direct:
        ctx.set_direct(True)
    slots = torch.arange(P.T, dtype=torch.int32, device="cuda")
    ctx.token_init(slots, dev_tensor(P.h0[0], P.dtype), 0)
    ctx.enqueue(0, slots, logits=torch.from_numpy(np.ascontiguousarray(P.tables[0][0, 0])).cuda())
    stats = ctx.run(retire_pass=passes)
    torch.cuda.synchronize()
    ctx.check()
    st = ctx.state()
    return ctx, stats, to_np(st["h"]), st


@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
def test_direct_top1_matches_oracle_and_pooled(dtype, monkeypatch):
    # the pooled run is compared bit for bit: keep it on the unsplit FFN (the fused cold kernel's
    # split reductions change fp32 summation order with the pick's shape)
    monkeypatch.setenv("AMOE_COLD", "0")
    P = Problem(**TOP1, dtype=dtype, seed=41)
    passes = 2
    ctx, stats, h, st = _run(P, True, passes)
    assert stats["token_layers"] == P.T * P.L * passes
    assert stats["legs"] == P.T * P.L * passes                    # K = 1: one leg per token-layer
    assert int(st["stats"][1]) == P.T                              # every token retired once
    W, SH = P.oracle_weights()
    ref, _ = drivers.sync_run(host_values(P.h0[0], dtype), P.logits, W, P.K, n_passes=passes, shared=SH,
                              dtype=dtype)
    # free-running over 2 layers x 2 passes at the contract's tolerances
    assert floored_err(h, ref) <= TOL[dtype]
    if dtype == "bf16":
        assert row_l2_err(h, ref) <= ROW_L2["bf16"]
    _, stats0, h0, _ = _run(P, False, passes)
    assert stats0["token_layers"] == stats["token_layers"]
    assert np.array_equal(h, h0)
    # the direct path launches no combine (its merge kernel replaces it): no more kernels per pick
    # than the pooled path, whose combine-ring snapshot runs inside the combine at G = 1
    assert stats["kernel_launches"] <= stats0["kernel_launches"]
    assert int(st["stats"][0]) == P.T * P.L * passes      # every merge counted on the home


def test_direct_requires_top1():
    from paper_2505_08944_b200.amoe import AmoeError
    P = Problem(L=1, E=8, K=2, S=0, d=128, ff=256, T=64, seed=3)
    ctx = P.make_ctx()
    with pytest.raises(AmoeError):
        ctx.set_direct(True)


def _gates(P, seed):
    from test_gpu_parity import _gate_params
    return _gate_params(P, seed)


def test_direct_top1_loopback_two_ranks(monkeypatch):
    """G = 2 on one GPU (loopback contexts, concurrent amoe_run threads): experts e mod 2, the
    router gate on every layer (each rank holds the gates). Direct forwarding stores remote
    homes' h / x / state over peer memory and scatters legs into the peer's rings. Result: legs
    crossed ranks, every token-layer merged once on its home, h against the oracle's gated run."""
    import threading
    monkeypatch.setenv("AMOE_COLD", "0")
    G, T = 2, 128
    P = Problem(L=2, E=8, K=1, S=0, d=128, ff=256, T=T, G=G, seed=43)
    gates, dev = _gates(P, 7)

    def run_ranks(direct=True):
        ctxs = [P.make_ctx(rank=r) for r in range(G)]
        ptrs = [c.ws.data_ptr() for c in ctxs]
        for c in ctxs:
            c.import_peers(ptrs)
            for l in range(P.L):
                c.set_gate(l, *dev[l])
            if direct:
                c.set_direct(True)
        streams = [torch.cuda.Stream() for _ in range(G)]
        for r, c in enumerate(ctxs):
            with torch.cuda.stream(streams[r]):
                slots = torch.arange(T, dtype=torch.int32, device="cuda")
                c.token_init(slots, dev_tensor(P.h0[r], "bf16"), 0)
                c.enqueue(0, slots)
        torch.cuda.synchronize()
        stats, errs = [None] * G, []

        def worker(r):
            try:
                with torch.cuda.stream(streams[r]):
                    stats[r] = ctxs[r].run(retire_pass=1, stream=streams[r])
            except Exception as e:   # pragma: no cover - reported below
                errs.append((r, e))

        th = [threading.Thread(target=worker, args=(r,)) for r in range(G)]
        for t in th:
            t.start()
        for t in th:
            t.join(timeout=120)
        assert not any(t.is_alive() for t in th), "amoe_run did not terminate"
        assert not errs, errs
        torch.cuda.synchronize()
        for c in ctxs:
            c.check()
        h = np.concatenate([to_np(c.state()["h"]) for c in ctxs])
        remote = sum(int(c.state()["stats"][3]) for c in ctxs)
        merged = [int(c.state()["stats"][0]) for c in ctxs]
        return h, stats, remote, merged

    h1, s1, rem1, merged1 = run_ranks(True)
    assert merged1 == [T * P.L] * G                 # each home counts its tokens' merges
    assert sum(s["token_layers"] for s in s1) == G * T * P.L
    assert rem1 > 0
    # against the oracle's gated synchronous run over the box's tokens (rows whose routing is not
    # decided by an fp32-sized logit gap; the direct merge computes the gate with CUDA-core fp32
    # dot products, the pooled combine on the tensor cores, so the two are compared via the oracle)
    from oracle import numerics as nx
    W, SH = P.oracle_weights()
    h0all = np.concatenate([host_values(P.h0[r], "bf16") for r in range(G)])
    ref, recs = drivers.sync_run(h0all, P.logits, W, P.K, n_passes=1, shared=SH, gates=gates, record=True)
    ok = np.ones(G * T, dtype=bool)
    for r, l in zip(recs, range(P.L)):
        zs = np.sort(nx.gate_logits(r["x"], *gates[l]).astype(np.float64), axis=1)[:, ::-1]
        ok &= (zs[:, 0] - zs[:, 1]) > 5e-3
    assert ok.mean() > 0.8
    assert floored_err(h1[ok], ref[ok]) <= TOL["bf16"]
