#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_cold.py -q -p no:cacheprovider -rf > gpurun_out/pytest_cold.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_cold.log
tail -15 gpurun_out/pytest_cold.log
for cfg in "deepseek 1 1" "deepseek 1 64" "deepseek 1 128" "deepseek 8 64" "mixtral 1 128" "mixtral 1 1"; do
  set -- $cfg
  AMOE_LIB=_ab/libamoe_ctrace.so timeout 120 python tools/cold_trace.py --shape $1 --experts $2 --n $3 2>&1 | tail -1
done | tee gpurun_out/cold_trace.log
timeout 900 python tools/cold_sweep.py --ns 1,16,128 --out gpurun_out/cold_sweep.json > gpurun_out/cold_sweep.log 2>&1; echo "sweep rc=$?"
cat gpurun_out/cold_sweep.log | python -c "
import sys,json
for l in sys.stdin:
    try: r=json.loads(l)
    except: print(l.strip()); continue
    print(r['shape'],r['experts'],r['n'],r['mode'],r['us'],r['frac'])"
