#!/usr/bin/env python
"""Scheduler ablation: Algorithm 1 "Defrag" vs MTFS vs FLFS, grouped per
layer vs the paper's single (layer, expert) pick, from two starting states, on one B200.

  wave   : every token enters layer 0 together (the bench's step; the wave stays consolidated)
  spread : token t starts at layer t mod L (the fragmented state re-batching exists for,
           PAPER.md L107-L114, L244) and runs closed-loop until pass R

Reports token-layers/s over the whole run (native amoe_run loop, CUDA events), scheduler picks,
(layer, expert) executions and the mean executed batch (legs per execution).

    python tools/sched_ablation.py [--config mixtral] [--passes 2] [--out profiles/r01_sched_ablation.json]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="mixtral")
    ap.add_argument("--passes", type=int, default=2)
    ap.add_argument("--T", type=int, default=0)
    ap.add_argument("--policies", default="defrag,mtfs,flfs,sync")
    ap.add_argument("--starts", default="wave,spread")
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    import numpy as np
    import torch
    import workload as wl
    from paper_2505_08944_b200 import amoe

    spec = wl.CONFIGS[args.config]
    L, E, K, S, d, ff = spec.L, spec.E, spec.K, spec.S, spec.d, spec.ff
    T = args.T or spec.T
    dev = torch.device("cuda", 0)
    cfg = amoe.make_config(L, E, K, S, d, ff, T)
    ctx = amoe.Context(cfg, device=dev)
    gen = torch.Generator(device=dev)
    gen.manual_seed(0)
    wts = []
    for l in range(L):
        for e in range(E + S):
            w1 = torch.empty(ff, d, dtype=torch.bfloat16, device=dev).normal_(0, d ** -0.5, generator=gen)
            w3 = torch.empty(ff, d, dtype=torch.bfloat16, device=dev).normal_(0, d ** -0.5, generator=gen)
            w2 = torch.empty(d, ff, dtype=torch.bfloat16, device=dev).normal_(0, ff ** -0.5, generator=gen)
            ctx.set_expert(l, e, w1, w3, w2)
            wts.append((w1, w3, w2))
    n_tab = 2
    table = torch.from_numpy(np.stack([wl.router_logits(0, L, T, E, zipf_s=spec.zipf_s, pass_idx=p)
                                       for p in range(n_tab)])).to(dev).contiguous()
    ctx.set_router(table)
    h0 = torch.from_numpy(wl.hidden0(0, T, d).view(np.int16)).view(torch.bfloat16).to(dev)
    slots = torch.arange(T, dtype=torch.int32, device=dev)

    def start(kind):
        ctx.token_init(slots, h0, 0)
        if kind == "wave":
            ctx.enqueue(0, slots, logits=table[0, 0])
            return T * L * args.passes
        lay = slots % L
        for l in range(L):
            sl = slots[lay == l].contiguous()
            ctx.enqueue(l, sl, logits=table[0, l][sl.long()].contiguous())
        return int(sum(L * args.passes - (t % L) for t in range(T)))

    rows = []
    for kind in args.starts.split(","):
        for policy in args.policies.split(","):
            if policy == "sync" and kind != "wave":
                continue            # lockstep layers need every token at the same layer
            for grouped in (True, False):
                # warm-up (same configuration, one pass)
                start(kind)
                ctx.run(retire_pass=1, policy=policy, grouped=grouped)
                torch.cuda.synchronize()
                expect = start(kind)
                torch.cuda.synchronize()
                ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                ev0.record()
                st = ctx.run(retire_pass=args.passes, policy=policy, grouped=grouped)
                ev1.record()
                torch.cuda.synchronize()
                ctx.check()
                ms = ev0.elapsed_time(ev1)
                assert st["token_layers"] == expect, (st, expect)
                r = {"config": args.config, "start": kind, "policy": policy, "grouped": grouped, "T": T,
                     "passes": args.passes, "token_layers": st["token_layers"], "ms": round(ms, 2),
                     "token_layers_per_s": round(st["token_layers"] / (ms / 1e3)),
                     "picks": st["picks"], "executions": st["queues_run"],
                     "mean_batch": round(st["legs"] / max(1, st["queues_run"]), 1),
                     "idle_polls": st["idle_polls"]}
                print(json.dumps(r), flush=True)
                rows.append(r)
    if args.out:
        with open(args.out, "w") as f:
            json.dump(rows, f, indent=1)


if __name__ == "__main__":
    main()
