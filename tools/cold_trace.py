#!/usr/bin/env python
"""Per-CTA timeline of the fused cold kernel (diagnostic build with -DAMOE_COLD_TRACE):

    python -m paper_2505_08944_b200.build --out _ab/libamoe_ctrace.so --flags=-DAMOE_COLD_TRACE
    AMOE_LIB=_ab/libamoe_ctrace.so python tools/cold_trace.py --shape deepseek --experts 1 --n 1

Stamps (globaltimer ns, relative to the earliest CTA entry): 0 entry, 1 producer past the grid
dependency, 2 producer done, 3 MMA issuer done, 4 first gather table loaded, 5 a gate/up split
reduced here (last arriver), 6 a down split reduced here, 7 gate/up epilogues done, 8 down
epilogues done, 11 exit. Prints min / median / max / count over CTAs.
"""
import argparse
import ctypes as C
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
NAMES = ["entry", "griddep", "producer_done", "mma_done", "gather_table", "redA_last", "redB_last", "epiA_done",
         "epiB_done", "W:mma_tempty", "-", "exit", "W:prod_empty", "W:mma_full", "W:gather_empty", "W:gather_cpasync"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="deepseek")
    ap.add_argument("--experts", type=int, default=1)
    ap.add_argument("--n", type=int, default=1)
    ap.add_argument("--reps", type=int, default=6)
    args = ap.parse_args()
    import torch
    from paper_2505_08944_b200 import amoe
    lib = amoe.load()
    if not hasattr(lib, "amoe_debug_cold_trace"):
        raise SystemExit("AMOE_LIB must point at a -DAMOE_COLD_TRACE build")
    d, ff = {"mixtral": (4096, 14336), "deepseek": (2048, 1408)}[args.shape]
    Gx, n = args.experts, args.n
    R = 4
    ctx = amoe.Context(amoe.make_config(R, Gx, 1, 0, d, ff, Gx * n))
    for l in range(R):
        for e in range(Gx):
            ctx.set_expert(l, e, torch.randn(ff, d, device="cuda", dtype=torch.bfloat16) * d ** -0.5,
                           torch.randn(ff, d, device="cuda", dtype=torch.bfloat16) * d ** -0.5,
                           torch.randn(d, ff, device="cuda", dtype=torch.bfloat16) * ff ** -0.5)
    nt = Gx * n
    slots = torch.arange(nt, dtype=torch.int32, device="cuda")
    idx = (torch.arange(nt, device="cuda", dtype=torch.int32) % Gx).view(nt, 1)
    h0 = torch.randn(nt, d, device="cuda", dtype=torch.bfloat16)
    gb = amoe.GroupBuffers(ctx, Gx * 128 + 256)
    buf = (C.c_ulonglong * (16 * 256))()
    for i in range(args.reps):
        l = i % R
        ctx.token_init(slots, h0)
        ctx.enqueue(l, slots, topk_idx=idx, topk_w=torch.ones(nt, 1, device="cuda"))
        gb.set_queues([(l, e) for e in range(Gx)], max_rows_hint=n)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        ctx.rebatch_ffn_forward(gb)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b)
    ctx.check()
    lib.amoe_debug_cold_trace(buf)
    tr = np.array(buf, dtype=np.uint64).reshape(16, 256).astype(np.int64)
    used = tr[0] > 0
    P = int(used.sum())
    t0 = tr[0][used].min()
    out = {"shape": args.shape, "experts": Gx, "n": n, "ctas": P, "event_us": round(ms * 1e3, 2), "points_us": {}}
    for i, name in enumerate(NAMES):
        v = tr[i][used]
        v = v[v > 0] - (0 if name.startswith("W:") else t0)
        if v.size:
            out["points_us"][name] = [round(float(v.min()) / 1e3, 2), round(float(np.median(v)) / 1e3, 2),
                                      round(float(v.max()) / 1e3, 2), int(v.size)]
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
