#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_cold.py -q -x -p no:cacheprovider 2>&1 | tail -2
for pf in 1 0; do
  AMOE_COLD_L2PF=$pf timeout 600 python tools/cold_sweep.py --shapes deepseek --groups 1,2,4,8 --ns 1,16,64 --modes cold > gpurun_out/l2pf_$pf.log 2>&1
done
python - <<'PY'
import json
t={}
for pf in (1,0):
    for l in open(f'gpurun_out/l2pf_{pf}.log'):
        try: r=json.loads(l)
        except: continue
        t.setdefault((r['shape'],r['experts'],r['n']),{})[pf]=(r['us'],r['frac'])
for k,v in t.items(): print(*k, 'pf1', v.get(1), 'pf0', v.get(0))
PY
