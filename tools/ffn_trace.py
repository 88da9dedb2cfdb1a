#!/usr/bin/env python
"""Per-CTA timeline of the CTA-pair FFN kernels (diagnostic build with -DAMOE_TRACE).

    AMOE_LIB=_ab/libamoe_trace.so python tools/ffn_trace.py --shape deepseek --n 16384

One (layer, expert) FFN of n re-batched tokens, launched a few times; the last gate/up and down
launches are traced: entry, setup done, first stage full, MMA done, pair end per CTA, and the MMA
issuer's time waiting on full stages / a free TMEM accumulator / the unit ring.
"""
import argparse
import ctypes as C
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from rebatch_sweep import SHAPES  # noqa: E402  (tools/ on sys.path when run as a script)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="deepseek")
    ap.add_argument("--n", type=int, default=16384)
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    import torch
    from paper_2505_08944_b200 import amoe
    lib = amoe.load()
    if not hasattr(lib, "amoe_debug_ffn_trace"):
        raise SystemExit("AMOE_LIB must point at a -DAMOE_TRACE build")
    d, ff, _ = SHAPES[args.shape]
    n = args.n
    ctx = amoe.Context(amoe.make_config(1, 1, 1, 0, d, ff, n))
    ctx.set_expert(0, 0, torch.randn(ff, d, device="cuda", dtype=torch.bfloat16) * d ** -0.5,
                   torch.randn(ff, d, device="cuda", dtype=torch.bfloat16) * d ** -0.5,
                   torch.randn(d, ff, device="cuda", dtype=torch.bfloat16) * ff ** -0.5)
    slots = torch.arange(n, dtype=torch.int32, device="cuda")
    ctx.token_init(slots, torch.randn(n, d, device="cuda", dtype=torch.bfloat16))
    ctx.enqueue(0, slots, topk_idx=torch.zeros(n, 1, dtype=torch.int32, device="cuda"),
                topk_w=torch.ones(n, 1, device="cuda"))
    gb = amoe.GroupBuffers(ctx, ((n + 255) // 256) * 256).set_queues([(0, 0)], max_rows_hint=n)
    ctx.rebatch(gb)
    for _ in range(5):
        ctx.expert_ffn(gb)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ctx.expert_ffn(gb)
    e1.record()
    torch.cuda.synchronize()
    buf = np.zeros((2, 8, 160), dtype=np.uint64)
    assert lib.amoe_debug_ffn_trace(buf.ctypes.data_as(C.POINTER(C.c_ulonglong))) == 0
    res = {"shape": args.shape, "n": n, "event_us_both": e0.elapsed_time(e1) * 1e3}
    for mi, mode in enumerate(("gateup", "down")):
        t = buf[mi].astype(np.int64)
        ncta = int((t[0] > 0).sum())          # CTAs launched (AMOE_TRACE_GRID may shrink the grid)
        t0 = t[0, :ncta].min()
        lead = np.arange(0, ncta, 2)
        foll = lead + 1
        end = t[3, foll]
        r = {
            "ctas": ncta,
            "span_us": float((end.max() - t0) / 1e3),
            "entry_spread_us": float((t[0, :ncta].max() - t0) / 1e3),
            "setup_us_median": float(np.median(t[1, :ncta] - t[0, :ncta]) / 1e3),
            "first_full_us_median": float(np.median(t[2, lead] - t[1, lead]) / 1e3),
            "first_full_us_max": float((t[2, lead] - t0).max() / 1e3),
            "mma_done_us_min": float((t[3, lead] - t0).min() / 1e3),
            "mma_done_us_median": float(np.median(t[3, lead] - t0) / 1e3),
            "mma_done_us_max": float((t[3, lead] - t0).max() / 1e3),
            "pair_end_minus_mma_done_us_median": float(np.median(end - t[3, lead]) / 1e3),
            "units_min": int(t[4, lead].min()), "units_max": int(t[4, lead].max()),
            "wait_full_us_median": float(np.median(t[5, lead]) / 1e3),
            "wait_tmem_us_median": float(np.median(t[6, lead]) / 1e3),
            "wait_ring_us_median": float(np.median(t[7, lead]) / 1e3),
        }
        res[mode] = r
    print(json.dumps(res, indent=1))
    if args.out:
        with open(args.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
