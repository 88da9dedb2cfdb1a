#!/usr/bin/env python
"""Per-launch table of an `ncu --metrics ... --csv` log (one line per kernel launch)."""
import csv
import sys

lines = open(sys.argv[1]).read().splitlines()
i = next(k for k, l in enumerate(lines) if l.startswith('"ID"'))
rows = list(csv.reader(lines[i:]))
h = rows[0]
ki, mi, vi, ii, ui = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID", "Metric Unit"))
d = {}
for r in rows[1:]:
    if len(r) == len(h):
        d.setdefault((int(r[ii]), r[ki].split("(")[0].replace("void ", "")), {})[r[mi]] = (r[vi], r[ui])
for (i, k), m in sorted(d.items()):
    print(i, k, "  ".join(f"{n.split('__')[1].split('.')[0]}={v}{u}" for n, (v, u) in m.items()))
