#!/usr/bin/env python
"""Open-loop serving on one B200 (throughput vs latency under
Poisson arrivals). Tokens arrive as a Poisson process of rate λ; the host loop admits every
arrived token (amoe_token_init + amoe_enqueue at layer 0) between scheduler steps
(amoe_run in stepping mode: one pick per call), each token runs one pass through the L layers
and retires. Per-token latency = device globaltimer at retirement - at admission
(AMOE_BUF_TOK_TIME); admission delay (arrival -> admitted by the host loop) reported apart.

    python tools/open_loop.py --config mixtral --N 8192 --rates 0.25,0.5,0.75,0.9 [--policies defrag,mtfs]

Rates are fractions of the closed-loop throughput of the same configuration measured first.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="mixtral")
    ap.add_argument("--N", type=int, default=8192, help="arrivals per measured rate (one slot each)")
    ap.add_argument("--rates", default="0.25,0.5,0.75,0.9")
    ap.add_argument("--policies", default="defrag,mtfs")
    ap.add_argument("--grouped", type=int, default=1)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    import numpy as np
    import torch
    import workload as wl
    from paper_2505_08944_b200 import amoe

    spec = wl.CONFIGS[args.config]
    L, E, K, S, d, ff, N = spec.L, spec.E, spec.K, spec.S, spec.d, spec.ff, args.N
    dev = torch.device("cuda", 0)
    ctx = amoe.Context(amoe.make_config(L, E, K, S, d, ff, N), device=dev)
    gen = torch.Generator(device=dev)
    gen.manual_seed(args.seed)
    keep = []
    for l in range(L):
        for e in range(E + S):
            w = (torch.empty(ff, d, dtype=torch.bfloat16, device=dev).normal_(0, d ** -0.5, generator=gen),
                 torch.empty(ff, d, dtype=torch.bfloat16, device=dev).normal_(0, d ** -0.5, generator=gen),
                 torch.empty(d, ff, dtype=torch.bfloat16, device=dev).normal_(0, ff ** -0.5, generator=gen))
            ctx.set_expert(l, e, *w)
            keep.append(w)
    table = torch.from_numpy(wl.router_logits(args.seed, L, N, E, zipf_s=spec.zipf_s)[None]).to(dev).contiguous()
    ctx.set_router(table)
    h0 = torch.from_numpy(wl.hidden0(args.seed, N, d).view(np.int16)).view(torch.bfloat16).to(dev)
    slots_all = torch.arange(N, dtype=torch.int32, device=dev)

    def closed_loop(policy):
        ctx.token_init(slots_all, h0, 0)
        ctx.enqueue(0, slots_all, logits=table[0, 0])
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ctx.run(retire_pass=1, policy=policy, grouped=bool(args.grouped))
        torch.cuda.synchronize()
        return N * L / (time.perf_counter() - t0)

    def open_loop(policy, rate_tl):
        lam = rate_tl / L                                   # token arrivals per second
        rng = np.random.default_rng(args.seed + 1)
        arrive = np.cumsum(rng.exponential(1.0 / lam, N))
        admitted_at = np.zeros(N)
        nxt = 0
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        while True:
            now = time.perf_counter() - t0
            hi = int(np.searchsorted(arrive, now, side="right"))
            if hi > nxt:
                sl = slots_all[nxt:hi]
                ctx.token_init(sl, h0[nxt:hi], 0)
                ctx.enqueue(0, sl, logits=table[0, 0][nxt:hi])
                admitted_at[nxt:hi] = time.perf_counter() - t0
                nxt = hi
            st = ctx.run(retire_pass=1, policy=policy, grouped=bool(args.grouped), max_picks=1)
            if nxt == N and st["picks"] == 0:
                torch.cuda.synchronize()
                if int(ctx.state()["stats"][1]) - retired0 >= N:
                    break
            elif st["picks"] == 0 and nxt < N:
                time.sleep(max(0.0, min(1e-4, arrive[nxt] - (time.perf_counter() - t0))))
        ctx.check()
        tt = ctx.state()["tok_time"].cpu().numpy().astype(np.float64)
        lat = (tt[:, 1] - tt[:, 0]) / 1e6                   # ms
        span = (tt[:, 1].max() - tt[:, 0].min()) / 1e9
        return {"offered_token_layers_per_s": rate_tl, "achieved_token_layers_per_s": N * L / span,
                "latency_ms_p50": float(np.percentile(lat, 50)), "latency_ms_p90": float(np.percentile(lat, 90)),
                "latency_ms_p99": float(np.percentile(lat, 99)),
                "admission_delay_ms_p99": float(np.percentile(1e3 * (admitted_at - arrive), 99))}

    rows = []
    for policy in args.policies.split(","):
        closed_loop(policy)                                  # warm-up
        cap = closed_loop(policy)
        for f in [float(x) for x in args.rates.split(",")]:
            retired0 = int(ctx.state()["stats"][1])
            r = open_loop(policy, f * cap)
            r.update(config=args.config, policy=policy, grouped=bool(args.grouped), N=N, closed_loop_capacity=cap,
                     load=f)
            print(json.dumps(r), flush=True)
            rows.append(r)
    if args.out:
        json.dump(rows, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
