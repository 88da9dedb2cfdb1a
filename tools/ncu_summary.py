#!/usr/bin/env python
"""Summarise ncu outputs into profiles/: a launch list (--metrics gpu__time_duration.sum pass)
and the key counters of a --set full capture.

    python tools/ncu_summary.py launches gpurun_out/launches.csv > profiles/rXX_launches.md
    python tools/ncu_summary.py full gpurun_out/prof.ncu-rep > profiles/rXX_ffn_full.md
"""
import collections
import csv
import io
import subprocess
import sys

FULL_METRICS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "launch__grid_size", "launch__cluster_dim_x",
    "launch__registers_per_thread", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_tc_scope_1cta.sum", "sm__inst_executed_pipe_tc_scope_2cta.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
]


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr, data = rows[hi], rows[hi + 1:]
    ki, mi, vi, ui = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    agg = collections.OrderedDict()
    dram = collections.defaultdict(float)
    unit = None
    for r in data:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].replace("void ", "")
        if r[mi] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            f = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(r[ui], 1)
            dram[name] += float(r[vi].replace(",", "")) * f
            continue
        if r[mi] != "gpu__time_duration.sum":
            continue
        unit = r[ui]
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += float(r[vi].replace(",", ""))
    scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}.get(unit, 1e-6)
    torch_like = ("distribution", "Fill", "elementwise", "arange", "die_probe", "spin_kernel", "reduce_kernel<")
    hot = {k: v for k, v in agg.items() if not any(t in k for t in torch_like) or "splitk" in k}
    tot = sum(v[1] for v in hot.values())
    print(f"| kernel | launches | total ms | mean us | share of libamoe time | DRAM MB per launch | DRAM GB/s |\n|---|---|---|---|---|---|---|")
    for k, (n, t) in sorted(hot.items(), key=lambda x: -x[1][1]):
        mb = dram.get(k, 0.0) / n / 1e6
        gbs = dram.get(k, 0.0) / (t * scale * 1e-3) / 1e9 if t else 0.0
        print(f"| `{k}` | {n} | {t * scale:.2f} | {1e3 * t * scale / n:.1f} | {100 * t / tot:.2f}% | {mb:.1f} | {gbs:.0f} |")
    other = {k: v for k, v in agg.items() if k not in hot}
    if other:
        print("\nNon-libamoe kernels in the same process (setup: weight init, arange):")
        for k, (n, t) in other.items():
            print(f"- `{k[:80]}` x{n}: {t * scale:.1f} ms")


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        print(f"### `{r[hdr.index('Kernel Name')]}`\n\n| metric | value | unit |\n|---|---|---|")
        for m in FULL_METRICS:
            if m in hdr:
                i = hdr.index(m)
                print(f"| {m} | {r[i]} | {units[i]} |")
        print()


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
