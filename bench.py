#!/usr/bin/env python
"""bench.py — MoE-layer tokens/s of the AEP expert hot path on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config mixtral|deepseek|tiny]
    python bench.py --impl reference ...      # the CPU oracle on the same workload (bounded sample)
    torchrun --nproc-per-node N bench.py --gpus N ...

A step is one decode pass of every in-flight token through all L expert layers (all §8(a) rows:
route + scatter into µ-queues, Algorithm-1 pick, re-batch gather, tcgen05 SwiGLU FFN, forward,
weighted combine + RMSNorm + relabel). Work per step = T_slots * L token-layers per GPU (weak
scaling: experts sharded e mod N, T_slots tokens homed per GPU). Inputs (hidden states, router
logits, weights) are resident in HBM before the timed region; the weights (90 GB for Mixtral)
are far larger than L2, so no flush is needed between steps.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "MoE-layer tokens/s"
UNIT = "token-layers/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="mixtral", choices=["mixtral", "deepseek", "tiny"])
    ap.add_argument("--policy", default="defrag_global", choices=["defrag", "mtfs", "flfs", "sync", "defrag_global"],
                    help="defrag_global = Algorithm 1 with the box-wide lookahead (identical to defrag on one "
                         "GPU; ahead of it at G > 1 in the G-rank emulation); sync = synchronous-EP baseline: "
                         "lockstep layers, box-wide barrier per layer")
    # Algorithm 1's lookahead (reading c11): W = 4, δ = 0.5 on one GPU; at G > 1
    # W = 8, δ = 1.0, the best of the G-rank emulation sweep (profiles/r02/g_emulate_sweep2.log:
    # Mixtral G = 4 1.20-1.23 M vs sync EP 1.14-1.16 M, G = 2 1.38 M vs 1.38-1.39 M)
    ap.add_argument("--W", type=int, default=None, help="Algorithm 1 lookahead depth (default 4; 8 at G > 1)")
    ap.add_argument("--delta", type=float, default=None, help="Algorithm 1 lookahead decay (default 0.5; 1.0 at G > 1)")
    ap.add_argument("--ungrouped", action="store_true", help="one (layer, expert) queue per launch")
    ap.add_argument("--T", type=int, default=0, help="override tokens in flight per GPU")
    ap.add_argument("--L", type=int, default=0, help="override layers (parity/debug only)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--router", default="table", choices=["table", "gate"],
                    help="table: synthetic Zipf logits (the paper's eval); gate: device router gate "
                         "x·Wgᵀ + per-layer Zipf log-prob bias computed in the combine (SURVEY.md f3)")
    ap.add_argument("--shift-every", type=int, default=1000,
                    help="skew epoch length in layer-steps (BASELINE.json configs[3]: 1000; reading c6): the "
                         "per-layer expert permutation is redrawn every that many layer traversals of the wave")
    ap.add_argument("--topk", type=int, default=0, help="override top-K (1: the paper's Top-1 routing, P:L463)")
    ap.add_argument("--direct", action="store_true",
                    help="top-1 direct forwarding (amoe_set_direct; needs --topk 1): the executing rank "
                         "merges and routes each token itself, no token pool / combine launch (SURVEY.md f3)")
    ap.add_argument("--skew", default="zipf", choices=["zipf", "exp"],
                    help="routing skew: Zipf s=1.2 (BASELINE.json) or the paper's exponential fit (λ=0.38)")
    args = ap.parse_args()
    if args.W is None:
        args.W = 8 if args.gpus > 1 else 4
    if args.delta is None:
        args.delta = 1.0 if args.gpus > 1 else 0.5
    return args


def FFN_KERNEL(d):
    """Name of the gate/up kernel the library launches (CTA pair unless d % 256 or AMOE_FFN_1CTA=1)."""
    if d % 256 == 0 and os.environ.get("AMOE_FFN_1CTA", "0") != "1":
        return "ffn_tc2_kernel<GATEUP> (tcgen05 cta_group::2 UMMA 256x256, fused SwiGLU)"
    return "ffn_tc_kernel<GATEUP> (tcgen05 UMMA 128x256, fused SwiGLU)"


def config_dict(spec, L, T, G, policy, grouped, skew="zipf", router="table", direct=False, shift_every=1000):
    """The workload description shared by both arms' JSON lines."""
    return {"workload": f"{spec.name}-shaped expert layers: L={L} E={spec.E} top-{spec.K} S={spec.S} d={spec.d} "
                        f"ff={spec.ff}, {T} tokens in flight per GPU, "
                        + (f"Zipf s={spec.zipf_s}" if skew == "zipf" else "exponential λ=0.38") + " routing",
            "experts_per_gpu": f"e mod {G}", "policy": policy, "grouped": grouped, "router": router,
            "l2": "inputs larger than L2 (resident weights >> 126 MB); no flush",
            "skew_shift_every_layer_steps": shift_every,
            "step": "one decode pass: every token through all L layers",
            "merge": "direct top-1 forwarding on the executing rank" if direct else "token pool + combine on the home"}


def peaks_bf16():
    """(burst, sustained, label): the driver-measured bf16 peaks, else the profiling guide's
    fallback (1.59 PFLOP/s burst, ~1.4 sustained under the power cap), labelled as such."""
    try:
        p = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return (float(p["bf16_tflops"]), float(p["bf16_tflops_sustained"]),
                "of measured: sustained bf16 cuBLAS (MEASURED_PEAKS.json)")
    except Exception:
        return 1590.0, 1400.0, "of fallback: 1.4 PFLOP/s sustained bf16 (B200_PROFILING.md; MEASURED_PEAKS.json absent)"


def peak_hbm():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]), "of measured"
    except Exception:
        return 6650.0, "of fallback (B200_PROFILING.md)"


def ncu_traffic(config, kernel, L, T):
    """DRAM bytes per launch of the dominant kernel from the committed `ncu --set full` summary,
    used only when the capture is of this kernel and workload (else null)."""
    try:
        rec = json.load(open(os.path.join(ROOT, "profiles", "ncu_summary.json"))).get(config, {})
    except Exception:
        return None
    if rec.get("kernel") != kernel.split(" ")[0] or rec.get("T") != T:
        return None
    return rec.get("ffn_gateup_dram_bytes_per_launch")


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    return ws, int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0"))


# ---------------------------------------------------------------------------------- clocks

class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 200 ms during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                       "-lms", "200", "-i", str(self.idx)], stdout=subprocess.PIPE,
                                      stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.p.terminate()
        out, _ = self.p.communicate(timeout=10)
        sm, smax, reasons, power = [], [], set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1])); smax.append(float(f[2])); power.append(float(f[3]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm), "power_w_max": max(power) if power else None}


# ---------------------------------------------------------------------------------- CPU oracle

_ORACLE_INPUTS = {}


def _oracle_inputs(spec, seed, max_tokens):
    """Layer-0 weights, logits and hidden states of the workload (generated once, not timed)."""
    import workload as wl
    key = (spec.name, seed, max_tokens)
    if key not in _ORACLE_INPUTS:
        W = [tuple(wl.f32_from_bf16_bits(a) for a in wl.expert_weights(seed, 0, e, spec.d, spec.ff))
             for e in range(spec.E)]
        SH = [tuple(wl.f32_from_bf16_bits(a) for a in wl.expert_weights(seed, 0, spec.E + j, spec.d, spec.ff))
              for j in range(spec.S)]
        z = wl.router_logits(seed, spec.L, min(spec.T, max_tokens), spec.E, layers=[0])[0]
        h = wl.f32_from_bf16_bits(wl.hidden0(seed, min(spec.T, max_tokens), spec.d))
        _ORACLE_INPUTS.clear()
        _ORACLE_INPUTS[key] = (W, SH, z, h)
    return _ORACLE_INPUTS[key]


def host_info():
    """The host the oracle ran on: CPU model, affinity cores, BLAS library and its threads."""
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    blas = None
    try:
        from threadpoolctl import threadpool_info
        for r in threadpool_info():
            if r.get("user_api") == "blas":
                blas = {"library": r.get("internal_api"), "version": r.get("version"),
                        "threads": r.get("num_threads"), "arch": r.get("architecture")}
                break
    except Exception:
        pass
    return {"cpu_model": model, "affinity_cores": len(os.sched_getaffinity(0)), "blas": blas}


def _limits(n):
    try:
        from threadpoolctl import threadpool_limits
        return threadpool_limits(limits=n)
    except Exception:  # pragma: no cover
        return None


def cpu_oracle_sample(spec, seed, budget_s=15.0, max_tokens=4096, threads=None):
    """Time the oracle (as it stands) on a bounded sample of the same workload: batches of
    tokens through layer 0 of the configuration (routing, SwiGLU experts, combine, RMSNorm).
    BLAS threads = the affinity cores (set explicitly, OpenBLAS oversubscribes
    by default)."""
    from oracle import numerics as nx
    cores = threads or len(os.sched_getaffinity(0))
    W, SH, z, h = _oracle_inputs(spec, seed, max_tokens)
    ctxm = _limits(cores)
    try:
        done, t0, batch = 0, time.perf_counter(), 64 if spec.d >= 2048 else 512
        while done < h.shape[0]:
            sl = slice(done, min(done + batch, h.shape[0]))
            nx.moe_layer(h[sl], z[sl], W, spec.K, SH, "bf16")
            done = sl.stop
            if time.perf_counter() - t0 > budget_s:
                break
        el = time.perf_counter() - t0
    finally:
        if ctxm is not None:
            ctxm.__exit__(None, None, None)
    return {"value": done / el, "unit": UNIT, "cores": cores, "threads": cores, "kind": "oracle",
            "sample": f"{done} tokens x layer 0 of the {spec.name} config (numpy float64 GEMMs, bf16 "
                      f"rounding), {el:.1f} s"}


def cpu_oracle_tiny_e2e(seed):
    """BASELINE.md §3's tiny-config oracle runs, end to end: the synchronous driver (fixed-batch
    EP) and the asynchronous µ-queue driver (Algorithm 1 over random interleavings), one pass of
    all 512 tokens through both layers, single BLAS thread (tiny GEMMs oversubscribe otherwise)."""
    import workload as wl
    from oracle import drivers
    spec = wl.CONFIGS["tiny"]
    W = [[tuple(wl.f32_from_bf16_bits(a) for a in wl.expert_weights(seed, l, e, spec.d, spec.ff))
          for e in range(spec.E)] for l in range(spec.L)]
    tab = wl.router_logits(seed, spec.L, spec.T, spec.E)
    h0 = wl.f32_from_bf16_bits(wl.hidden0(seed, spec.T, spec.d))
    out = {}
    ctxm = _limits(1)
    try:
        for name in ("sync", "async"):
            t0 = time.perf_counter()
            if name == "sync":
                drivers.sync_run(h0, lambda p, l: tab[l], W, spec.K, n_passes=1)
            else:
                drivers.async_run(h0, lambda p, l: tab[l], W, spec.K, G=1, T=spec.T, n_passes=1, seed=seed)
            el = time.perf_counter() - t0
            out[name] = {"value": spec.T * spec.L / el, "unit": UNIT, "threads": 1,
                         "sample": f"tiny config, {spec.T} tokens x {spec.L} layers, {el:.2f} s"}
    finally:
        if ctxm is not None:
            ctxm.__exit__(None, None, None)
    return out


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:   # rank 0 alone runs the CPU oracle; the other ranks exit without work
        return
    import workload as wl
    spec = wl.CONFIGS[args.config]
    # each step = one bounded sample (<= 128 tokens through layer 0, <= 10 s of oracle work);
    # inputs are generated once before the warm-up (not timed)
    for _ in range(args.warmup):
        cpu_oracle_sample(spec, args.seed, budget_s=3.0, max_tokens=128)
    vals = []
    t0 = time.perf_counter()
    for _ in range(args.steps):
        r = cpu_oracle_sample(spec, args.seed, budget_s=10.0, max_tokens=128)
        vals.append(r["value"])
    el = time.perf_counter() - t0
    value = statistics.median(vals)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * el / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64-accum/bf16-storage",
            "data": "synthetic (seeded workload generator)",
            "config": config_dict(spec, spec.L, spec.T, args.gpus, args.policy, not args.ungrouped),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": r["cores"], "kind": "oracle",
                             "sample": r["sample"], "host": host_info()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------------- our arm

def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import numpy as np
    import torch
    import torch.distributed as dist

    import workload as wl
    from paper_2505_08944_b200 import amoe
    from paper_2505_08944_b200 import dist as D

    G, rank, local = D.env()
    assert G == args.gpus, f"--gpus {args.gpus} but WORLD_SIZE {G}"
    # AMOE_DIST_BACKEND=gloo: ranks may share a GPU (local rank mod device count) — the N > 1
    # path exercised on a one-GPU box; the data path is the same (peer workspaces via IPC)
    backend = os.environ.get("AMOE_DIST_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if G > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    cdev = dev if backend == "nccl" else "cpu"       # device of the timing / stall reductions
    spec = wl.CONFIGS[args.config]
    if args.topk:
        import dataclasses
        spec = dataclasses.replace(spec, K=args.topk)
    L = args.L or spec.L
    T = args.T or spec.T
    E, K, S, d, ff = spec.E, spec.K, spec.S, spec.d, spec.ff
    cfg = amoe.make_config(L, E, K, S, d, ff, T, G=G, rank=rank, dtype="bf16")
    nbytes = amoe.workspace_bytes(cfg)
    if G > 1:
        ws, ptrs = D.peer_workspace(nbytes + 256, dev)
        ctx = amoe.Context(cfg, workspace=ws, device=dev)
        ctx.import_peers(ptrs)
    else:
        ctx = amoe.Context(cfg, device=dev)

    # resident inputs: weights of hosted experts (seeded, N(0,1/d), N(0,1/ff)), router tables, h0
    gen = torch.Generator(device=dev)
    gen.manual_seed(args.seed * 1000 + rank)
    wts = []
    for l in range(L):
        for e in D.hosted_experts(E, S, G, rank):
            w1 = torch.empty(ff, d, dtype=torch.bfloat16, device=dev).normal_(0, d ** -0.5, generator=gen)
            w3 = torch.empty(ff, d, dtype=torch.bfloat16, device=dev).normal_(0, d ** -0.5, generator=gen)
            w2 = torch.empty(d, ff, dtype=torch.bfloat16, device=dev).normal_(0, ff ** -0.5, generator=gen)
            ctx.set_expert(l, e, w1, w3, w2)
            wts.append((w1, w3, w2))
    # router tables: one per pass when the skew epoch shifts within the run (every pass then
    # carries its own epoch's permutations), else two alternating passes of epoch 0
    n_pass = args.warmup + args.steps
    shifting = args.shift_every < n_pass * L
    n_tab = n_pass if shifting else 2
    tables_host = [wl.router_logits(args.seed, L, T, E, zipf_s=spec.zipf_s, pass_idx=p, token_offset=rank * T,
                                    skew=args.skew, shift_every=args.shift_every)
                   for p in range(n_tab)]
    epochs = sorted({wl.skew_epoch(p, l, L, args.shift_every) for p in range(args.warmup, n_pass) for l in range(L)})
    table = torch.from_numpy(np.stack(tables_host)).to(dev).contiguous()
    ctx.set_router(table)
    if args.direct:
        ctx.set_direct(True)
    gate_w = []
    if args.router == "gate":
        for l in range(L):
            wg = torch.empty(E, d, dtype=torch.bfloat16, device=dev).normal_(0, d ** -0.5, generator=gen)
            perm = torch.from_numpy(wl.layer_perm(args.seed, l, 0, E).argsort()).to(dev)
            bias = torch.from_numpy(np.log(wl.skew_probs(E, args.skew, spec.zipf_s))).float().to(dev)[perm].contiguous()
            ctx.set_gate(l, wg, bias)
            gate_w.append((wg, bias))
    h0 = torch.from_numpy(wl.hidden0(args.seed, T, d, token_offset=rank * T).view(np.int16)).view(
        torch.bfloat16).to(dev)
    slots = torch.arange(T, dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream()
    policy, grouped = args.policy, not args.ungrouped

    def step(p):
        ctx.token_init(slots, h0, p)
        if args.router == "gate":
            ctx.enqueue(0, slots)
        else:
            ctx.enqueue(0, slots, logits=table[p % n_tab, 0])
        return ctx.run(retire_pass=p + 1, policy=policy, W=args.W, delta=args.delta, grouped=grouped)

    barrier = D.barrier
    # every rank must have created (zeroed) its workspace before any rank pushes legs into it
    torch.cuda.synchronize()
    barrier()

    for w in range(args.warmup):
        step(w)
    torch.cuda.synchronize()
    ctx.check()

    # ------------------------------------------------------------------ timed region
    clocks = ClockSampler(local if "CUDA_VISIBLE_DEVICES" not in os.environ else
                          int(os.environ["CUDA_VISIBLE_DEVICES"].split(",")[local]))
    # per-stage CUDA events (the roofline's kernel times and the schedule's execution log) inside
    # the timed region; AMOE_BENCH_STAGE_EVENTS=0 times the step without them (A/B of their cost)
    stage_events = os.environ.get("AMOE_BENCH_STAGE_EVENTS", "1") != "0"
    ctx.profile_enable(stage_events)
    barrier()
    torch.cuda.synchronize()
    clocks.start()
    launches0 = ctx.launch_count()
    remote0 = int(ctx.state()["stats"][3])
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    runs = []
    for k in range(args.steps):
        runs.append(step(args.warmup + k))
    ev1.record(stream)
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    launches = ctx.launch_count() - launches0
    remote_legs = int(ctx.state()["stats"][3]) - remote0     # legs this rank ran for another home
    ms = ev0.elapsed_time(ev1)
    prof = ctx.profile_read()
    execs = ctx.exec_log()
    ctx.profile_enable(False)
    ctx.check()
    token_layers = sum(r["token_layers"] for r in runs)
    legs = sum(r["legs"] for r in runs)
    # per-GPU stall: host wall time of scheduler polls that found nothing of this rank's to run
    stall = D.gather_values([sum(r["idle_ns"] for r in runs) / max(1, sum(r["wall_ns"] for r in runs)),
                             sum(r["barriers"] for r in runs)], device=cdev)
    ms, (token_layers, legs) = D.reduce_timing(ms, [token_layers, legs], device=cdev)
    assert token_layers == G * T * L * args.steps, (token_layers, G * T * L * args.steps)
    value = token_layers / (ms / 1e3)

    # roofline of the dominant kernel (tcgen05 gate/up + SwiGLU GEMM): algorithmic FLOPs per
    # launch = 4 d ff n (n = legs in the launch) over its CUDA-event duration
    peak_burst, peak_sust, peak_kind = peaks_bf16()
    my_legs = sum(r["legs"] for r in runs)
    gu_ms, gu_n = prof["ffn_gateup"]
    dn_ms, dn_n = prof["ffn_down"]
    gu_tflops = 4.0 * d * ff * my_legs / (gu_ms / 1e3) / 1e12 if gu_ms else None
    dn_tflops = 2.0 * d * ff * my_legs / (dn_ms / 1e3) / 1e12 if dn_ms else None
    traffic = ncu_traffic(args.config, FFN_KERNEL(d), L, T)
    stage_ms = {k: round(v[0], 3) for k, v in prof.items()}
    # HBM-bound steps (SURVEY.md §8(d) per-unit bytes): combine+RMSNorm+route/scatter per
    # token-layer = (K+S)·d·2 pool + 3·d·2 (h in, h out, x out) + E·4 logits; re-batch per leg =
    # 2·d·2 (x row in, tile row out)
    hbm_pk, hbm_kind = peak_hbm()
    my_tl = sum(r["token_layers"] for r in runs)
    hbm = {}
    # AMOE_CP_GATHER=1 (one GPU, CTA-pair FFN): the re-batch gather runs inside the gate/up
    # producer (cp.async copies of the legs' x rows); "rebatch" is then the drain
    fused_gather = (G == 1 and os.environ.get("AMOE_CP_GATHER", "0") == "1" and d % 256 == 0
                    and os.environ.get("AMOE_FFN_1CTA", "0") != "1" and not args.direct)
    for name, nbytes, ms_ in (("combine", my_tl * ((K + S) * d * 2 + 3 * d * 2 + E * 4), prof["combine"][0]),
                              ("rebatch", my_legs * 4 * d, prof["rebatch"][0])):
        if name == "rebatch" and fused_gather:
            hbm[name] = {"fused": "gather inside the gate/up GEMM's producer warp (cp.async A rows from x)",
                         "drain_ms": round(ms_, 3), "gather_kernel_bytes": 0}
            continue
        if ms_:
            gbs = nbytes / (ms_ / 1e3) / 1e9
            hbm[name] = {"achieved": round(gbs, 1), "peak": hbm_pk, "unit": "GB/s", "frac": round(gbs / hbm_pk, 3),
                         "peak_kind": hbm_kind, "algorithmic_bytes": int(nbytes)}
    step_ms = ms / args.steps

    # schedule-conditional roofline: every logged execution of n legs costs
    # max(6·d·ff·n / F_pk, (6·d·ff + 4·n·d) / BW) (weights streamed once + tile in/out), plus the
    # combine's algorithmic bytes / BW; t_ideal = all FLOPs / F_pk (charges fragmentation too).
    f_pk = peak_sust * 1e12
    bw = hbm_pk * 1e9
    t_exec = sum(max(6.0 * d * ff * n / f_pk, (6.0 * d * ff + 4.0 * n * d) / bw) for _, _, n in execs)
    t_act = my_tl * ((K + S) * d * 2 + 3 * d * 2 + E * 4) / bw
    t_ideal = 6.0 * d * ff * my_legs / f_pk
    per_rank = D.gather_values([1e3 * (t_exec + t_act), 1e3 * t_ideal], device=cdev)
    t_roof_ms = max(v[0] for v in per_rank)
    t_ideal_ms = max(v[1] for v in per_rank)
    hist = {}
    for _, _, n in execs:
        b = 1 << max(0, int(n).bit_length() - 1)
        hist[b] = hist.get(b, 0) + 1
    step_roof = {"t_roof_ms": round(t_roof_ms, 3), "t_ideal_ms": round(t_ideal_ms, 3), "measured_ms": round(ms, 3),
                 "frac_of_schedule_roofline": round(t_roof_ms / ms, 4), "frac_of_ideal": round(t_ideal_ms / ms, 4),
                 "peaks": f"{peak_sust} TFLOP/s ({peak_kind.split(':')[0]}), {hbm_pk} GB/s ({hbm_kind})",
                 "executions_rank0": len(execs),
                 "mean_legs_per_execution_rank0": round(my_legs / max(1, len(execs)), 1),
                 "legs_per_execution_hist_rank0": {f">={k}": v for k, v in sorted(hist.items())}}

    # NVLink term: a leg run on a rank other than its token's home moves the
    # x row home -> owner (the gather's peer load, d·2 B) and the output row owner -> home (the
    # down epilogue's peer store, d·2 B) plus its 16-B ring entry; per rank and direction the
    # larger of the two, against 900 GB/s; combined with the step roofline two ways (overlap:
    # max, BASELINE.json's literal "plus": sum). Analytic need for uniform placement: 2·K·d·2·(G−1)/G
    # bytes per homed token-layer (both directions).
    per_rank_nv = D.gather_values([remote_legs, my_legs], device=cdev)
    rem_max = max(v[0] for v in per_rank_nv)
    nv_dir_bytes = rem_max * (d * 2 + 16) / args.steps             # per step, per direction, busiest rank
    nv_peak = 900.0
    t_nv_ms = nv_dir_bytes / (nv_peak * 1e9) * 1e3 * args.steps
    legs_all = [v[1] for v in per_rank_nv]
    share = max(legs_all) / max(1, sum(legs_all))
    nvlink = {"bytes_per_step_per_direction_busiest_rank": int(nv_dir_bytes),
              "gbs_per_direction": round(nv_dir_bytes / (step_ms / 1e3) / 1e9, 2), "peak": nv_peak, "unit": "GB/s",
              "frac": round(nv_dir_bytes / (step_ms / 1e3) / 1e9 / nv_peak, 5),
              "remote_legs_per_rank": [int(v[0]) for v in per_rank_nv],
              "measured_bytes_per_token_layer": round(2 * sum(v[0] for v in per_rank_nv) * (d * 2 + 16)
                                                      / max(1, G * T * L * args.steps), 1),
              "analytic_bytes_per_token_layer_uniform": round(2 * K * d * 2 * (G - 1) / G, 1),
              "t_nvlink_ms": round(t_nv_ms, 3),
              "step_roofline_max_ms": round(max(t_roof_ms, t_nv_ms), 3),
              "step_roofline_sum_ms": round(t_roof_ms + t_nv_ms, 3),
              "frac_of_step_roofline_max": round(max(t_roof_ms, t_nv_ms) / ms, 4),
              "frac_of_step_roofline_sum": round((t_roof_ms + t_nv_ms) / ms, 4)}
    placement = {"legs_per_rank": [int(x) for x in legs_all], "hottest_rank_share": round(share, 4),
                 "cap_speedup_vs_1gpu": round(1.0 / share, 3) if share else None,
                 "note": "speedup over one GPU is bounded by 1 / the hottest rank's share of the legs (SURVEY.md §8(e))"}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": G, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": step_ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "bf16", "data": "synthetic (seeded Zipf s=1.2 routing, random-init bf16 weights)",
        "config": dict(config_dict(spec, L, T, G, policy, grouped, args.skew, args.router, args.direct, args.shift_every),
                       lookahead={"W": args.W, "delta": args.delta}),
        "gpu_launches": int(launches),
        "die_map_sms": list(amoe.die_info()),
        "clocks": clk,
        "stall": {"idle_frac_per_rank": [round(v[0], 4) for v in stall], "layer_barriers": int(stall[0][1]),
                  "busy_frac_rank0": round(sum(v[0] for v in prof.values()) / ms, 4) if ms else None,
                  "definition": "time a rank's scheduler found no runnable queue / its amoe_run wall time"},
        "roofline": {"bound": "tensor", "kernel": FFN_KERNEL(d),
                     "achieved": gu_tflops, "peak": peak_sust, "unit": "TFLOP/s",
                     "frac": (gu_tflops / peak_sust) if gu_tflops else None,
                     "peak_kind": peak_kind,
                     "frac_of_burst": (gu_tflops / peak_burst) if gu_tflops else None,
                     "traffic": traffic,
                     "algorithmic": "4*d*ff FLOP per leg (gate+up), legs per launch = drained tokens",
                     "down_kernel_tflops": dn_tflops,
                     "ffn_tflops": (6.0 * d * ff * my_legs / ((gu_ms + dn_ms) / 1e3) / 1e12) if gu_ms else None,
                     "stage_ms_total": stage_ms,
                     "stage_launches": {k: v[1] for k, v in prof.items()},
                     "hbm_kernels": hbm,
                     "step": step_roof,
                     "nvlink": nvlink},
        "placement": placement,
        "skew_epochs_in_timed_region": epochs,
    }

    # ------------------------------------------------------------------ end to end (host buffers)
    if not args.no_e2e:
        h0_host = h0.cpu().pin_memory()
        hout = torch.empty_like(h0_host).pin_memory()
        rt_host = [torch.from_numpy(t).pin_memory() for t in tables_host]
        for w in range(1):
            ctx.pass_host(h0_host, hout, rt_host[w % n_tab], pass_idx=w, policy=policy, W=args.W, delta=args.delta,
                          grouped=grouped)
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for k in range(args.steps):
            ctx.pass_host(h0_host, hout, rt_host[k % n_tab], pass_idx=k, policy=policy, W=args.W, delta=args.delta,
                          grouped=grouped)
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        ems, _ = D.reduce_timing(e0.elapsed_time(e1), [], device=cdev)
        line["e2e"] = {"value": G * T * L * args.steps / (ems / 1e3), "unit": UNIT,
                       "h2d_bytes_per_step": int(h0_host.numel() * 2 + rt_host[0].numel() * 4),
                       "d2h_bytes_per_step": int(hout.numel() * 2),
                       "api": "amoe_pass_host (C ABI, pinned host buffers)"}

    # ------------------------------------------------------------------ CPU oracle baseline
    if rank == 0 and G == 1 and not args.no_cpu_baseline:
        cb = cpu_oracle_sample(spec, args.seed)
        cb["host"] = host_info()
        # BASELINE.md §3's other oracle samples, reported beside the headline one
        extra = {}
        try:
            extra["tiny_e2e"] = cpu_oracle_tiny_e2e(args.seed)
            other = "deepseek" if spec.name == "mixtral" else "mixtral"
            ds = cpu_oracle_sample(wl.CONFIGS[other], args.seed, budget_s=6.0, max_tokens=2048)
            extra[f"{other}_layer0"] = ds
        except Exception as e:  # pragma: no cover - reported, never fatal
            extra["error"] = repr(e)
        cb["other_samples"] = extra
        line["cpu_baseline"] = cb

    if rank == 0:
        print(json.dumps(line), flush=True)
    if G > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
