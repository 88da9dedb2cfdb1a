"""Workload for compute-sanitizer (tools/sanitize.sh): the tiny config end to end through amoe_run
(grouped Algorithm 1, 2 passes; the 1-CTA tcgen05 kernels since d % 256 != 0), a d = 256 variant
on the CTA-pair kernels, and two loopback ranks (G = 2) running amoe_run concurrently on their
own streams (peer rings, system-scope atomics, fused forward into the peer's pool)."""
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


def loopback(G=2):
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
            out[r] = ctxs[r].run(retire_pass=2, stream=streams[r])

    th = [threading.Thread(target=w, args=(r,)) for r in range(G)]
    [t.start() for t in th]
    [t.join() for t in th]
    torch.cuda.synchronize()
    for c in ctxs:
        c.check()
    print(f"loopback G={G}: {[o['token_layers'] for o in out]}", flush=True)


if __name__ == "__main__":
    from paper_2505_08944_b200 import build
    build.build()
    what = sys.argv[1] if len(sys.argv) > 1 else "all"
    if what in ("all", "single"):
        single(128)
        single(256)
    if what in ("all", "loopback"):
        loopback(2)
