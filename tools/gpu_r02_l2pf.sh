#!/bin/bash
# fused cold kernel: L2 prefetch distance A/B (AMOE_COLD_L2PF = 0 / 1 / 2 ring depths ahead)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for rep in a b; do
  for pf in 0 1 2; do
    AMOE_COLD_L2PF=$pf timeout 300 python tools/cold_sweep.py --shapes deepseek,mixtral --groups 1,8 --ns 1,16,32,64 --modes cold --iters 10 > gpurun_out/l2pf_${pf}_$rep.log 2>&1
  done
done
AMOE_COLD_L2PF=1 timeout 300 python -m pytest tests/test_gpu_cold.py -x -q > gpurun_out/pytest_cold_pf.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_cold_pf.log
tail -2 gpurun_out/pytest_cold_pf.log
python - <<'PY'
import json,glob
t={}
for f in sorted(glob.glob('gpurun_out/l2pf_*.log')):
    pf=f.split('_')[2]
    for l in open(f):
        try: r=json.loads(l)
        except: continue
        t.setdefault((r['shape'],r['experts'],r['n']),{}).setdefault(pf,[]).append(r['us'])
for k,v in sorted(t.items()): print(*k, {p: [round(x,1) for x in u] for p,u in sorted(v.items())})
PY
