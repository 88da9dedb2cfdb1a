#!/usr/bin/env python
"""FFN kernel microbenchmark under the B200 power cap: one grouped layer (all experts), drained
once, then amoe_expert_ffn looped for a fixed wall time per variant while nvidia-smi samples SM
clock and power. Reports TFLOP/s, clock, power and TFLOP/s per W per variant.

    python tools/ffn_micro.py [--config mixtral|deepseek] [--T 16384] [--secs 4]
        [--variants "1cta:2048,2cta:2048,2cta:8192"]
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def sample_start():
    return subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits",
                             "-lms", "100", "-i", "0"], stdout=subprocess.PIPE, text=True)


def sample_stop(p):
    time.sleep(0.15)
    p.terminate()
    out, _ = p.communicate()
    sm, pw = [], []
    for line in out.strip().splitlines():
        try:
            a, b = line.split(",")
            sm.append(float(a)); pw.append(float(b))
        except ValueError:
            pass
    return (statistics.median(sm) if sm else None, statistics.median(pw) if pw else None)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="mixtral")
    ap.add_argument("--T", type=int, default=0)
    ap.add_argument("--secs", type=float, default=4.0)
    ap.add_argument("--variants", default="1cta:2048,2cta:2048,2cta:4096,2cta:8192")
    args = ap.parse_args()
    import numpy as np
    import torch
    import workload as wl
    from paper_2505_08944_b200 import amoe
    spec = wl.CONFIGS[args.config]
    T = args.T or spec.T
    E, K, S, d, ff = spec.E, spec.K, spec.S, spec.d, spec.ff
    cfg = amoe.make_config(1, E, K, S, d, ff, T)
    ctx = amoe.Context(cfg)
    for e in range(E + S):
        ctx.set_expert(0, e, torch.randn(ff, d, device="cuda", dtype=torch.bfloat16) * d ** -0.5,
                       torch.randn(ff, d, device="cuda", dtype=torch.bfloat16) * d ** -0.5,
                       torch.randn(d, ff, device="cuda", dtype=torch.bfloat16) * ff ** -0.5)
    tab = torch.from_numpy(wl.router_logits(0, 1, T, E)[None]).cuda().contiguous()
    ctx.set_router(tab)
    slots = torch.arange(T, dtype=torch.int32, device="cuda")
    h0 = torch.randn(T, d, device="cuda", dtype=torch.bfloat16)
    ctx.token_init(slots, h0)
    ctx.enqueue(0, slots, logits=tab[0, 0])
    gb = amoe.GroupBuffers(ctx, T * K + T * S + 128 * (E + S))
    gb.set_queues([(0, e) for e in range(E + S)])
    ctx.rebatch(gb)
    torch.cuda.synchronize()
    legs = int(gb.info()[0].sum())
    flop = 6.0 * d * ff * legs
    res = []
    for v in args.variants.split(","):
        kind, rows = v.split(":")
        if kind == "cublas":
            # library reference on the same FLOPs: [legs x d] @ [d x 2ff] then [legs x ff] @ [ff x d]
            X = torch.randn(legs, d, device="cuda", dtype=torch.bfloat16)
            W13 = torch.randn(2 * ff, d, device="cuda", dtype=torch.bfloat16)
            A = torch.randn(legs, ff, device="cuda", dtype=torch.bfloat16)
            W2 = torch.randn(d, ff, device="cuda", dtype=torch.bfloat16)
            for _ in range(3):
                X @ W13.t(); A @ W2.t()
            torch.cuda.synchronize()
            p = sample_start()
            t0, n = time.time(), 0
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev0.record()
            while time.time() - t0 < args.secs:
                for _ in range(8):
                    X @ W13.t(); A @ W2.t()
                n += 8
                torch.cuda.synchronize()
            ev1.record()
            torch.cuda.synchronize()
            sm, pw = sample_stop(p)
            ms = ev0.elapsed_time(ev1) / n
            tf = flop / (ms / 1e3) / 1e12
            r = {"variant": v, "legs": legs, "ms_per_ffn": round(ms, 3), "tflops": round(tf, 1), "sm_mhz": sm,
                 "power_w": pw, "tflops_per_w": round(tf / pw, 3) if pw else None,
                 "tflop_per_mhz": round(tf / sm, 3) if sm else None}
            print(json.dumps(r), flush=True)
            del X, W13, A, W2
            continue
        os.environ["AMOE_FFN_1CTA"] = "1" if kind == "1cta" else "0"
        os.environ["AMOE_GROUP_M"] = rows
        for _ in range(3):
            ctx.expert_ffn(gb)
        torch.cuda.synchronize()
        ctx.profile_enable(True)
        p = sample_start()
        t0 = time.time()
        n = 0
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        while time.time() - t0 < args.secs:
            for _ in range(8):
                ctx.expert_ffn(gb)
            n += 8
            torch.cuda.synchronize()
        ev1.record()
        torch.cuda.synchronize()
        sm, pw = sample_stop(p)
        prof = ctx.profile_read()
        ctx.profile_enable(False)
        ms = ev0.elapsed_time(ev1) / n
        tf = flop / (ms / 1e3) / 1e12
        r = {"variant": v, "legs": legs, "ms_per_ffn": round(ms, 3), "tflops": round(tf, 1),
             "gateup_ms": round(prof["ffn_gateup"][0] / n, 3), "down_ms": round(prof["ffn_down"][0] / n, 3),
             "sm_mhz": sm, "power_w": pw, "tflops_per_w": round(tf / pw, 3) if pw else None,
             "tflop_per_mhz": round(tf / sm, 3) if sm else None}
        print(json.dumps(r), flush=True)
        res.append(r)


if __name__ == "__main__":
    main()
