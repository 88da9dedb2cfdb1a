#!/bin/bash
# cold v2: parity tests, device-only sweep, per-CTA trace
mkdir -p gpurun_out _ab
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_cold.py -q -x -p no:cacheprovider -rf > gpurun_out/pytest_cold.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_cold.log
tail -15 gpurun_out/pytest_cold.log
timeout 600 python tools/cold_sweep.py --ns 1,16,64,128 --out gpurun_out/cold_sweep3.json > gpurun_out/cold_sweep3.log 2>&1; echo "sweep rc=$?"
python - <<'PY'
import json
for l in open('gpurun_out/cold_sweep3.log'):
    try: r=json.loads(l)
    except: print(l.strip()[:200]); continue
    print(r['shape'],r['experts'],r['n'],r['mode'],r['us'],r['frac'])
PY
python -m paper_2505_08944_b200.build --out _ab/libamoe_ctrace.so --flags=-DAMOE_COLD_TRACE > gpurun_out/build_ctrace.log 2>&1
for cfg in "deepseek 1 1" "deepseek 1 128" "deepseek 8 64" "mixtral 1 1" "mixtral 1 128"; do
  set -- $cfg
  AMOE_COLD=1 AMOE_LIB=_ab/libamoe_ctrace.so timeout 120 python tools/cold_trace.py --shape $1 --experts $2 --n $3 2>&1 | tail -1
done | tee gpurun_out/cold_trace2.log
