#!/usr/bin/env python
"""G ranks emulated on ONE GPU: G contexts in one process, each on its own stream and host
thread, each with persistent grids sized for num_sms / G SMs (AMOE_NUM_SMS), so they co-run on
roughly disjoint halves of the chip. Experts are sharded e mod G, legs cross ranks through the
peer-mapped workspaces exactly as on G GPUs. What differs from G real GPUs: the ranks share
one HBM, one L2 and one power budget, and the hardware may place any CTA anywhere.

    python tools/g_emulate.py --config mixtral --policy defrag --G 2 --steps 3

Prints one JSON line: token-layers/s over all ranks (host wall time, device-synchronised, around
the G concurrent amoe_run calls of each step), per-rank idle fraction, layer barriers.
"""
import argparse
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="mixtral")
    ap.add_argument("--policy", default="defrag")
    ap.add_argument("--W", type=int, default=4, help="Algorithm 1 lookahead depth")
    ap.add_argument("--delta", type=float, default=0.5, help="Algorithm 1 lookahead decay")
    ap.add_argument("--G", type=int, default=2)
    ap.add_argument("--L", type=int, default=0)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--skew", default="zipf", help="router skew: zipf (s from the config) or exp")
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    import torch
    import workload as wl
    from paper_2505_08944_b200 import amoe
    from paper_2505_08944_b200 import dist as D

    spec = wl.CONFIGS[args.config]
    G = args.G
    L = args.L or spec.L
    T, E, K, S, d, ff = spec.T, spec.E, spec.K, spec.S, spec.d, spec.ff
    dev = torch.device("cuda", 0)
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    os.environ["AMOE_NUM_SMS"] = str((sms // G) & ~1)
    ctxs, keep, tables, h0s = [], [], [], []
    gen = torch.Generator(device=dev)
    for r in range(G):
        cfg = amoe.make_config(L, E, K, S, d, ff, T, G=G, rank=r, dtype="bf16")
        c = amoe.Context(cfg, device=dev)
        gen.manual_seed(args.seed * 1000 + r)
        for l in range(L):
            for e in D.hosted_experts(E, S, G, r):
                w = (torch.empty(ff, d, dtype=torch.bfloat16, device=dev).normal_(0, d ** -0.5, generator=gen),
                     torch.empty(ff, d, dtype=torch.bfloat16, device=dev).normal_(0, d ** -0.5, generator=gen),
                     torch.empty(d, ff, dtype=torch.bfloat16, device=dev).normal_(0, ff ** -0.5, generator=gen))
                c.set_expert(l, e, *w)
                keep.append(w)
        tab = torch.from_numpy(np.stack([wl.router_logits(args.seed, L, T, E, zipf_s=spec.zipf_s, pass_idx=p,
                                                          token_offset=r * T, skew=args.skew)
                                          for p in range(2)])).to(dev)
        c.set_router(tab)
        tables.append(tab)
        h0s.append(torch.from_numpy(wl.hidden0(args.seed, T, d, token_offset=r * T).view(np.int16)).view(
            torch.bfloat16).to(dev))
        ctxs.append(c)
    ptrs = [c.ws.data_ptr() for c in ctxs]
    for c in ctxs:
        c.import_peers(ptrs)
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream() for _ in range(G)]
    slots = torch.arange(T, dtype=torch.int32, device=dev)

    def step(p):
        for r, c in enumerate(ctxs):
            with torch.cuda.stream(streams[r]):
                c.token_init(slots, h0s[r], p)
                c.enqueue(0, slots, logits=tables[r][p % 2, 0])
        torch.cuda.synchronize()
        stats, errs = [None] * G, []

        def worker(r):
            try:
                stats[r] = ctxs[r].run(retire_pass=p + 1, policy=args.policy, W=args.W, delta=args.delta,
                                       stream=streams[r])
            except Exception as e:  # reported below
                errs.append((r, repr(e)))
        th = [threading.Thread(target=worker, args=(r,)) for r in range(G)]
        t0 = time.perf_counter()
        for t in th:
            t.start()
        for t in th:
            t.join(timeout=600)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        if errs or any(t.is_alive() for t in th):
            raise SystemExit(f"rank failure: {errs}")
        return dt, stats

    for w in range(args.warmup):
        step(w)
    total, runs = 0.0, []
    for k in range(args.steps):
        dt, st = step(args.warmup + k)
        total += dt
        runs.append(st)
    for c in ctxs:
        c.check()
    tl = sum(s["token_layers"] for st in runs for s in st)
    assert tl == G * T * L * args.steps, (tl, G * T * L * args.steps)
    idle = [sum(st[r]["idle_ns"] for st in runs) / max(1, sum(st[r]["wall_ns"] for st in runs)) for r in range(G)]
    line = {"tool": "g_emulate", "config": args.config, "policy": args.policy, "skew": args.skew, "W": args.W, "delta": args.delta, "G": G,
            "sms_per_rank": int(os.environ["AMOE_NUM_SMS"]), "L": L, "T_per_rank": T, "steps": args.steps,
            "value": tl / total, "unit": "token-layers/s (host wall, device-synced)",
            "ms_per_step": 1e3 * total / args.steps, "idle_frac_per_rank": [round(x, 4) for x in idle],
            "layer_barriers": [sum(st[r]["barriers"] for st in runs) for r in range(G)],
            "picks_per_rank": [sum(st[r]["picks"] for st in runs) for r in range(G)]}
    print(json.dumps(line), flush=True)
    if args.out:
        with open(args.out, "w") as f:
            json.dump(line, f, indent=1)


if __name__ == "__main__":
    main()
