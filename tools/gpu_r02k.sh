#!/bin/bash
mkdir -p gpurun_out _ab
python -m paper_2505_08944_b200.build --out _ab/libamoe_ctrace.so --flags=-DAMOE_COLD_TRACE > gpurun_out/build_ctrace.log 2>&1 &
python -m paper_2505_08944_b200.build --out _ab/libamoe_ng.so --flags="-DAMOE_COLD_TRACE -DAMOE_COLD_NOGATHER" > gpurun_out/build_ng.log 2>&1 &
python -m paper_2505_08944_b200.build --out _ab/libamoe_np.so --flags="-DAMOE_COLD_TRACE -DAMOE_COLD_NOMMA" > gpurun_out/build_np.log 2>&1 &
wait
for lib in ctrace ng np; do
for cfg in "mixtral 1 128" "deepseek 8 64"; do
  set -- $cfg
  echo -n "$lib "; AMOE_COLD=1 AMOE_LIB=_ab/libamoe_$lib.so timeout 120 python tools/cold_trace.py --shape $1 --experts $2 --n $3 2>&1 | tail -1
done; done > gpurun_out/cold_trace6.log
python - <<'PY'
import json
for l in open('gpurun_out/cold_trace6.log'):
    lib,_,js=l.partition(' ')
    try: r=json.loads(js)
    except: print(l.strip()[:300]); continue
    p=r['points_us']
    print(lib, r['shape'],r['experts'],r['n'],' '.join(f"{k}={v[1]}/{v[2]}" for k,v in p.items() if v[1]>=0 and k in ('epiA_done','exit','W:mma_full','W:prod_empty','W:gather_empty','W:mma_tempty')))
PY
