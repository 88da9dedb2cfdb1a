"""Workload for compute-sanitizer (tools/sanitize.sh): the tiny config end to end through amoe_run
(grouped Algorithm 1, 2 passes; the 1-CTA tcgen05 kernels since d % 256 != 0), a d = 256 variant
on the CTA-pair kernels, and two loopback ranks (G = 2) running amoe_run concurrently on their
own streams (peer rings, system-scope atomics, fused forward into the peer's pool). Round 2 adds
`cold` (the fused cold-pick kernel, forced, grouped and single-queue picks, top-6 + 2 shared),
`direct` (top-1 direct forwarding) and `global` (loopback G = 2 with the box-wide Algorithm 1)."""
import os
import sys
import threading

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]

import numpy as np  # noqa: E402
import torch  # noqa: E402

from parity_util import Problem, dev_tensor  # noqa: E402


def admit(ctx, P, rank=0):
    slots = torch.arange(P.T, dtype=torch.int32, device="cuda")
    ctx.token_init(slots, dev_tensor(P.h0[rank], "bf16"), 0)
    ctx.enqueue(0, slots, logits=torch.from_numpy(np.ascontiguousarray(P.tables[rank][0, 0])).cuda())


def single(d):
    P = Problem(L=2, E=8, K=2, S=0, d=d, ff=256, T=512, seed=1)
    ctx = P.make_ctx()
    admit(ctx, P)
    st = ctx.run(retire_pass=2)
    torch.cuda.synchronize()
    ctx.check()
    print(f"single d={d}: {st['token_layers']} token-layers", flush=True)


def loopback(G=2, policy="defrag"):
    T = 128
    P = Problem(L=2, E=8, K=2, S=0, d=256, ff=256, T=T, G=G, seed=2)
    ctxs = [P.make_ctx(rank=r) for r in range(G)]
    ptrs = [c.ws.data_ptr() for c in ctxs]
    for c in ctxs:
        c.import_peers(ptrs)
    streams = [torch.cuda.Stream() for _ in range(G)]
    for r, c in enumerate(ctxs):
        with torch.cuda.stream(streams[r]):
            admit(c, P, r)
    torch.cuda.synchronize()
    out = [None] * G

    def w(r):
        with torch.cuda.stream(streams[r]):
            out[r] = ctxs[r].run(retire_pass=2, policy=policy, stream=streams[r])

    th = [threading.Thread(target=w, args=(r,)) for r in range(G)]
    [t.start() for t in th]
    [t.join() for t in th]
    torch.cuda.synchronize()
    for c in ctxs:
        c.check()
    print(f"loopback G={G} {policy}: {[o['token_layers'] for o in out]}", flush=True)


def cold():
    os.environ["AMOE_COLD"] = "1"
    try:
        for grouped in (True, False):
            P = Problem(L=2, E=16, K=6, S=2, d=256, ff=256, T=48, seed=3)
            ctx = P.make_ctx()
            admit(ctx, P)
            st = ctx.run(retire_pass=2, policy="defrag" if grouped else "mtfs", grouped=grouped)
            torch.cuda.synchronize()
            ctx.check()
            print(f"cold grouped={grouped}: {st['token_layers']} token-layers", flush=True)
    finally:
        os.environ.pop("AMOE_COLD")


def direct():
    P = Problem(L=2, E=8, K=1, S=0, d=256, ff=256, T=256, seed=4)
    ctx = P.make_ctx()
    ctx.set_direct(True)
    admit(ctx, P)
    st = ctx.run(retire_pass=2)
    torch.cuda.synchronize()
    ctx.check()
    print(f"direct K=1: {st['token_layers']} token-layers", flush=True)


if __name__ == "__main__":
    from paper_2505_08944_b200 import build
    build.build()
    what = sys.argv[1] if len(sys.argv) > 1 else "all"
    if what in ("all", "single"):
        single(128)
        single(256)
    if what in ("all", "loopback"):
        loopback(2)
    if what in ("all", "cold"):
        cold()
    if what in ("all", "direct"):
        direct()
    if what in ("all", "global"):
        loopback(2, "defrag_global")
