#!/bin/bash
mkdir -p gpurun_out _ab
python -m paper_2505_08944_b200.build --out _ab/libamoe_ctrace.so --flags=-DAMOE_COLD_TRACE > gpurun_out/build_ctrace.log 2>&1
for cfg in "mixtral 1 128" "mixtral 1 64" "deepseek 8 128" "deepseek 1 128"; do
  set -- $cfg
  AMOE_COLD=1 AMOE_LIB=_ab/libamoe_ctrace.so timeout 120 python tools/cold_trace.py --shape $1 --experts $2 --n $3 2>&1 | tail -1
done > gpurun_out/cold_trace5.log
python - <<'PY'
import json
for l in open('gpurun_out/cold_trace5.log'):
    try: r=json.loads(l)
    except: print(l.strip()[:300]); continue
    p=r['points_us']
    print(r['shape'],r['experts'],r['n'],'ctas',r['ctas'],' '.join(f"{k}={v[1]}/{v[2]}" for k,v in p.items() if v[1]>=0))
PY
