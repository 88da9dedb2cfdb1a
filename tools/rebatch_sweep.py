#!/usr/bin/env python
"""Re-batch size sweep (BASELINE.json configs[4]): one (layer, expert) SwiGLU FFN re-batched to n
tokens, n = 1..4096, Mixtral- and DeepSeek-shaped, on one B200 — the cold (HBM-bound weight
streaming) to hot (tensor-bound) roofline curve behind the paper's Fig. 3 (PAPER.md L107-L114:
"increasing batch size increases throughput almost linearly until the batch size of 128").

Each measurement rotates over R distinct layers' weights so L2 (126 MB) never holds the expert:
Mixtral 352 MB per expert (R = 4), DeepSeek 17.3 MB (R = 32). Timed with CUDA events around
`amoe_expert_ffn` (gate/up + SwiGLU + down), after warm-up.

    python tools/rebatch_sweep.py [--shapes mixtral,deepseek] [--out profiles/r01_rebatch_sweep.json]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

NS = sorted({1, 2, 4, 8, 16, 24, 32, 48, 64, 96, 128, 192, 256, 320, 384, 512, 1024, 2048, 4096})
SHAPES = {"mixtral": (4096, 14336, 4), "deepseek": (2048, 1408, 32),
          # diagnostics: the DeepSeek width with 2x / 4x the FFN width (longer K in the down GEMM)
          "deepseek_ff2x": (2048, 2816, 16), "deepseek_ff4x": (2048, 5632, 8)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", default="mixtral,deepseek")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--out", default="")
    ap.add_argument("--ns", default="", help="comma-separated subset of n values")
    ap.add_argument("--grouped", type=int, default=0,
                    help="also measure G distinct experts with n tokens each in ONE grouped launch "
                         "(what the Algorithm-1 grouped pick executes for cold layers)")
    args = ap.parse_args()
    import torch
    from paper_2505_08944_b200 import amoe
    global NS
    if args.ns:
        NS = sorted(int(x) for x in args.ns.split(","))
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    hbm = peaks.get("hbm_gbs", 6650.0) * 1e9
    tc = peaks.get("bf16_tflops", 1590.0) * 1e12
    results = []
    for shape in args.shapes.split(","):
        d, ff, R = SHAPES[shape]
        nmax = max(NS)
        cfg = amoe.make_config(R, 1, 1, 0, d, ff, nmax)
        ctx = amoe.Context(cfg)
        for l in range(R):
            ctx.set_expert(l, 0, torch.randn(ff, d, device="cuda", dtype=torch.bfloat16) * d ** -0.5,
                           torch.randn(ff, d, device="cuda", dtype=torch.bfloat16) * d ** -0.5,
                           torch.randn(d, ff, device="cuda", dtype=torch.bfloat16) * ff ** -0.5)
        h0 = torch.randn(nmax, d, device="cuda", dtype=torch.bfloat16)
        for n in NS:
            slots = torch.arange(n, dtype=torch.int32, device="cuda")
            gbs = []
            for l in range(R):
                ctx.token_init(slots, h0[:n])
                ctx.enqueue(l, slots, topk_idx=torch.zeros(n, 1, dtype=torch.int32, device="cuda"),
                            topk_w=torch.ones(n, 1, device="cuda"))
                gb = amoe.GroupBuffers(ctx, ((n + 255) // 256) * 256).set_queues([(l, 0)], max_rows_hint=n)
                ctx.rebatch(gb)
                gbs.append(gb)
            torch.cuda.synchronize()
            for gb in gbs:
                ctx.expert_ffn(gb)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(args.iters):
                for gb in gbs:
                    ctx.expert_ffn(gb)
            e1.record()
            torch.cuda.synchronize()
            t = e0.elapsed_time(e1) / 1e3 / (args.iters * R)
            flop = 6.0 * d * ff * n
            wbytes = 6.0 * d * ff
            roof = max(flop / tc, (wbytes + 4.0 * n * d + 4.0 * n * ff) / hbm)
            r = {"shape": shape, "n": n, "us": round(t * 1e6, 2), "tflops": round(flop / t / 1e12, 2),
                 "weight_gbs": round(wbytes / t / 1e9, 1), "roofline_us": round(roof * 1e6, 2),
                 "frac_of_roofline": round(roof / t, 3), "bound": "tensor" if flop / tc > wbytes / hbm else "hbm"}
            print(json.dumps(r), flush=True)
            results.append(r)
            del gbs
        ctx.close()
        torch.cuda.empty_cache()
        if args.grouped:
            Gx = args.grouped
            cfg = amoe.make_config(2, Gx, 1, 0, d, ff, Gx * 256)
            ctx = amoe.Context(cfg)
            for l in range(2):
                for e in range(Gx):
                    ctx.set_expert(l, e, torch.randn(ff, d, device="cuda", dtype=torch.bfloat16) * d ** -0.5,
                                   torch.randn(ff, d, device="cuda", dtype=torch.bfloat16) * d ** -0.5,
                                   torch.randn(d, ff, device="cuda", dtype=torch.bfloat16) * ff ** -0.5)
            h0 = torch.randn(Gx * 256, d, device="cuda", dtype=torch.bfloat16)
            for n in [x for x in NS if x <= 256]:
                nt = n * Gx
                slots = torch.arange(nt, dtype=torch.int32, device="cuda")
                idx = (torch.arange(nt, device="cuda", dtype=torch.int32) % Gx).view(nt, 1)
                gbs = []
                for l in range(2):
                    ctx.token_init(slots, h0[:nt])
                    ctx.enqueue(l, slots, topk_idx=idx, topk_w=torch.ones(nt, 1, device="cuda"))
                    gb = amoe.GroupBuffers(ctx, Gx * ((n + 255) // 256) * 256).set_queues(
                        [(l, e) for e in range(Gx)], max_rows_hint=n)
                    ctx.rebatch(gb)
                    gbs.append(gb)
                for gb in gbs:
                    ctx.expert_ffn(gb)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(args.iters):
                    for gb in gbs:
                        ctx.expert_ffn(gb)
                e1.record()
                torch.cuda.synchronize()
                t = e0.elapsed_time(e1) / 1e3 / (args.iters * 2)
                flop = 6.0 * d * ff * nt
                wbytes = 6.0 * d * ff * Gx
                roof = max(flop / tc, (wbytes + 4.0 * nt * d + 4.0 * nt * ff) / hbm)
                r = {"shape": shape, "grouped_experts": Gx, "n": n, "us": round(t * 1e6, 2),
                     "tflops": round(flop / t / 1e12, 2), "weight_gbs": round(wbytes / t / 1e9, 1),
                     "roofline_us": round(roof * 1e6, 2), "frac_of_roofline": round(roof / t, 3),
                     "bound": "tensor" if flop / tc > wbytes / hbm else "hbm"}
                print(json.dumps(r), flush=True)
                results.append(r)
                del gbs
            ctx.close()
            torch.cuda.empty_cache()
    if args.out:
        json.dump({"peaks": {"hbm_gbs": hbm / 1e9, "bf16_tflops": tc / 1e12}, "rows": results},
                  open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
