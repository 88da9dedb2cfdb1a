#!/bin/bash
# cold v2 quick loop: parity tests, sweep, trace
mkdir -p gpurun_out _ab
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_cold.py -q -x -p no:cacheprovider -rf > gpurun_out/pytest_cold.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_cold.log
tail -3 gpurun_out/pytest_cold.log
timeout 600 python tools/cold_sweep.py --ns ${NS:-1,16,64,128} --modes ${MODES:-cold} --out gpurun_out/cold_sweep4.json > gpurun_out/cold_sweep4.log 2>&1; echo "sweep rc=$?"
python - <<'PY'
import json
for l in open('gpurun_out/cold_sweep4.log'):
    try: r=json.loads(l)
    except: print(l.strip()[:200]); continue
    print(r['shape'],r['experts'],r['n'],r['mode'],r['us'],r['frac'])
PY
python -m paper_2505_08944_b200.build --out _ab/libamoe_ctrace.so --flags=-DAMOE_COLD_TRACE > gpurun_out/build_ctrace.log 2>&1
for cfg in ${TRACE_CFGS:-"deepseek 1 1" "deepseek 8 1" "deepseek 8 64" "mixtral 1 1" "mixtral 8 1"}; do
  set -- $cfg
  AMOE_COLD=1 AMOE_LIB=_ab/libamoe_ctrace.so timeout 120 python tools/cold_trace.py --shape $1 --experts $2 --n $3 2>&1 | tail -1
done > gpurun_out/cold_trace4.log
python - <<'PY'
import json
for l in open('gpurun_out/cold_trace4.log'):
    try: r=json.loads(l)
    except: print(l.strip()[:300]); continue
    p=r['points_us']
    print(r['shape'],r['experts'],r['n'],' '.join(f"{k}={v[1]}/{v[2]}" for k,v in p.items() if v[1]>=0))
PY
