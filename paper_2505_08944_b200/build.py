"""Build libamoe.so in-tree with nvcc for sm_100a (no GPU needed; nvcc cross-compiles).

    python -m paper_2505_08944_b200.build [--force] [--verbose]
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "lib")
LIB = os.path.join(LIBDIR, "libamoe.so")
SOURCES = ["api.cu", "k_tokens.cu", "k_queue.cu", "k_ffn_tc.cu", "k_ffn_cold.cu", "k_ffn_simt.cu", "scheduler.cpp"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-O3", "-Xptxas", "-v",
    "-I", os.path.join(ROOT, "include"), "-I", CSRC,
]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "amoe.h")]
    return any(os.path.getmtime(p) > t for p in deps)


def build(force: bool = False, verbose: bool = False, out: str | None = None, extra=()) -> str:
    """Compile every source for sm_100a and link libamoe.so (in-tree unless `out`); `extra` adds
    nvcc flags (diagnostic variants, e.g. -DAMOE_COLD_TRACE, built into their own object dir)."""
    if out is None and not extra and not force and not _stale():
        return LIB
    lib = out or LIB
    os.makedirs(os.path.dirname(os.path.abspath(lib)), exist_ok=True)
    objdir = os.path.join(LIBDIR, "obj") if out is None else os.path.abspath(lib) + ".obj"
    os.makedirs(objdir, exist_ok=True)
    objs = []
    procs = []
    for src in SOURCES:
        obj = os.path.join(objdir, os.path.splitext(src)[0] + ".o")
        cmd = [NVCC, *FLAGS, *extra, "-c", os.path.join(CSRC, src), "-o", obj]
        if src.endswith(".cpp"):
            cmd = [NVCC, "-std=c++17", "-O3", "-Xcompiler", "-fPIC", "-I", os.path.join(ROOT, "include"),
                   "-c", os.path.join(CSRC, src), "-o", obj]
        procs.append((src, cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
        objs.append(obj)
    for src, cmd, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{' '.join(cmd)}\n{out}")
        if verbose:
            print(f"--- {src}\n{out}")
        with open(os.path.join(objdir, src + ".ptxas.txt"), "w") as f:
            # registers / spills / smem per kernel; compile times dropped (the report stays stable)
            f.write("".join(l for l in out.splitlines(True) if "Compile time" not in l))
    link = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler", "-fPIC",
            *objs, "-o", lib + ".tmp"]
    r = subprocess.run(link, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(lib + ".tmp", lib)
    return lib


if __name__ == "__main__":
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    ap.add_argument("--out", default=None, help="build a variant library here (not the in-tree one)")
    ap.add_argument("--flags", default="", help="extra nvcc flags, space separated")
    a = ap.parse_args()
    print(build(force=a.force, verbose=a.verbose, out=a.out, extra=tuple(a.flags.split())))
