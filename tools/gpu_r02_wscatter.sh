#!/bin/bash
# combine: per-warp leg scatter (in-tree) vs the CTA-wide scatter behind a block barrier
# (_ab/libamoe_head.so) and warp scatter without the prologue prefetch (_ab/libamoe_ws.so), bench stage times alternating; + the parity tests on the new build
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_replay.py -x -q > gpurun_out/pytest_ws.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ws.log
for rep in a b; do
  for lib in new head ws; do
    if [ $lib = new ]; then unset AMOE_LIB; else export AMOE_LIB=_ab/libamoe_$lib.so; fi
    timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/ws_mixtral_${lib}_$rep.json 2>> gpurun_out/ws.err
    timeout 300 python bench.py --config deepseek --no-cpu-baseline --no-e2e > gpurun_out/ws_deepseek_${lib}_$rep.json 2>> gpurun_out/ws.err
  done
done
unset AMOE_LIB
tail -2 gpurun_out/pytest_ws.log; tail -2 gpurun_out/ws.err
for f in gpurun_out/ws_*.json; do python - "$f" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r=d['roofline']
    print(sys.argv[1].split('/')[-1], round(d['value']), d['clocks']['sm_mhz'], 'combine', r['stage_ms_total']['combine'], r['hbm_kernels']['combine']['frac'], 'step', r['step']['frac_of_schedule_roofline'])
except Exception as e: print(sys.argv[1], 'ERR', e)
PY
done
