#!/usr/bin/env python
"""Cold-expert sweep of the whole executor step (a4 drain + gather, a5/a6 SwiGLU expert, a7 forward
into the home pools) — `amoe_rebatch_ffn_forward` — for Gx experts of one layer with n legs each,
Mixtral- and DeepSeek-shaped, on one B200 (BASELINE.json configs[4]).

Each call is timed alone with CUDA events on its stream (the re-enqueue of the legs between calls
is outside the events); weights rotate over R layers so L2 (126 MB) never holds them. The HBM
roofline of one call is (6·d·ff weights + 2·n·d token rows in + 2·n·d rows out per expert) / BW,
the tensor roofline 6·d·ff·n / peak; `frac` = max of the two / measured. AMOE_COLD=1 (default)
(mode "cold") takes the fused one-launch cold kernel (amoe_execute_cold, n <= 128, the queue
heads tracked here as the scheduler would); mode "classic" the four-kernel path.

    python tools/cold_sweep.py [--shapes mixtral,deepseek] [--groups 1,8] [--ns 1,16,64,128,256,384]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

SHAPES = {"mixtral": (4096, 14336), "deepseek": (2048, 1408)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", default="mixtral,deepseek")
    ap.add_argument("--groups", default="1,8")
    ap.add_argument("--ns", default="1,8,16,32,64,96,128,192,256,320,384,512")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--modes", default="cold,classic")
    ap.add_argument("--out", default="")
    ap.add_argument("--sleep-cycles", type=int, default=400000)
    args = ap.parse_args()
    import torch
    from paper_2505_08944_b200 import amoe
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    hbm = peaks.get("hbm_gbs", 6536.4) * 1e9
    tc = peaks.get("bf16_tflops", 1632.4) * 1e12
    ns = [int(x) for x in args.ns.split(",")]
    rows = []
    for shape in args.shapes.split(","):
        d, ff = SHAPES[shape]
        for Gx in (int(x) for x in args.groups.split(",")):
            wbytes_expert = 6.0 * d * ff
            R = max(2, int(4 * 126e6 // (wbytes_expert * Gx)) + 1)     # >= 4x L2 of distinct weights
            R = min(R, 64)
            nmax = max(ns)
            cfg = amoe.make_config(R, Gx, 1, 0, d, ff, Gx * nmax)
            ctx = amoe.Context(cfg)
            gen = torch.Generator(device="cuda")
            gen.manual_seed(0)
            for l in range(R):
                for e in range(Gx):
                    ctx.set_expert(l, e, torch.empty(ff, d, device="cuda", dtype=torch.bfloat16).normal_(0, d ** -0.5, generator=gen),
                                   torch.empty(ff, d, device="cuda", dtype=torch.bfloat16).normal_(0, d ** -0.5, generator=gen),
                                   torch.empty(d, ff, device="cuda", dtype=torch.bfloat16).normal_(0, ff ** -0.5, generator=gen))
            h0 = torch.randn(Gx * nmax, d, device="cuda", dtype=torch.bfloat16)
            gbs = [amoe.GroupBuffers(ctx, Gx * ((nmax + 255) // 256) * 256 + 256) for _ in range(R)]
            heads = [0] * R                    # consumer head of every queue of layer l (all advance together)
            for n in ns:
                nt = n * Gx
                slots = torch.arange(nt, dtype=torch.int32, device="cuda")
                idx = (torch.arange(nt, device="cuda", dtype=torch.int32) % Gx).view(nt, 1)
                wts = torch.ones(nt, 1, device="cuda")
                for mode in args.modes.split(","):
                    os.environ["AMOE_COLD"] = "1" if mode == "cold" else "0"
                    if mode == "cold" and n > 128:
                        continue
                    for g, l in zip(gbs, range(R)):
                        g.set_queues([(l, e) for e in range(Gx)], max_rows_hint=n)
                    evs = []
                    stream = torch.cuda.current_stream()
                    for i in range(args.iters + 2):
                        l = i % R
                        ctx.token_init(slots, h0[:nt])
                        ctx.enqueue(l, slots, topk_idx=idx, topk_w=wts)
                        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        # keep the stream busy while the host issues the call, so the events bracket
                        # device time only (not ctypes marshalling / launch latency of an idle GPU)
                        torch.cuda._sleep(args.sleep_cycles)
                        a.record(stream)
                        if mode == "cold":
                            # the scheduler's decision made explicit: each queue's head and depth
                            ctx.execute_cold(gbs[l], [heads[l]] * Gx, [n] * Gx)
                        else:
                            ctx.rebatch_ffn_forward(gbs[l])
                        heads[l] += n
                        b.record(stream)
                        if i >= 2:
                            evs.append((a, b))
                    torch.cuda.synchronize()
                    ctx.check()
                    t = sum(a.elapsed_time(b) for a, b in evs) / len(evs) / 1e3
                    flop = 6.0 * d * ff * nt
                    byts = wbytes_expert * Gx + 4.0 * nt * d
                    roof = max(flop / tc, byts / hbm)
                    r = {"shape": shape, "experts": Gx, "n": n, "mode": mode, "us": round(t * 1e6, 2),
                         "weight_gbs": round(wbytes_expert * Gx / t / 1e9, 1), "roofline_us": round(roof * 1e6, 2),
                         "frac": round(roof / t, 3), "bound": "tensor" if flop / tc > byts / hbm else "hbm",
                         "path": "cold fused (1 launch)" if (mode == "cold" and n <= 128) else "drain+gather+gateup+down",
                         "kakb": os.environ.get("AMOE_COLD_KAKB", "auto")}
                    print(json.dumps(r), flush=True)
                    rows.append(r)
            ctx.close()
            del gbs
            torch.cuda.empty_cache()
    if args.out:
        json.dump({"peaks": {"hbm_gbs": hbm / 1e9, "bf16_tflops": tc / 1e12},
                   "what": "amoe_rebatch_ffn_forward per call (drain, gather, SwiGLU expert, forward), CUDA events",
                   "rows": rows}, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
