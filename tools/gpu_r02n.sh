#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for rk in 64 160 512 2048; do
  AMOE_COLD_RED_KB=$rk timeout 300 python tools/cold_sweep.py --ns 16,32,64,128 --modes cold > gpurun_out/cold_rk_$rk.log 2>&1
done
timeout 300 python tools/cold_sweep.py --ns 16,32,64,128 --modes classic > gpurun_out/cold_rk_classic.log 2>&1
python - <<'PY'
import json,glob,collections
t=collections.defaultdict(dict)
for f in sorted(glob.glob('gpurun_out/cold_rk_*.log')):
    tag=f.split('_')[-1][:-4]
    for l in open(f):
        try: r=json.loads(l)
        except: continue
        t[(r['shape'],r['experts'],r['n'])][tag]=r['us']
tags=['64','160','512','2048','classic']
print('shape E n', *tags)
for k,v in t.items(): print(*k, *[v.get(x,'-') for x in tags])
PY
