#!/usr/bin/env python
"""Registers / spills per kernel from the build's saved `ptxas -v` output.
    python tools/ptxas_regs.py paper_2505_08944_b200/lib/obj/k_tokens.cu.ptxas.txt [substring]"""
import re
import subprocess
import sys

cur = None
for line in open(sys.argv[1]):
    m = re.search(r"Compiling entry function '(\w+)'", line)
    if m:
        cur = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
        spill = ""
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and cur:
        spill = f"spill st/ld {m.group(1)}/{m.group(2)}"
    m = re.search(r"Used (\d+) registers", line)
    if m and cur:
        if len(sys.argv) < 3 or sys.argv[2] in cur:
            print(f"{m.group(1):>4} regs  {spill:24s} {cur[:110]}")
        cur = None
