#!/bin/bash
# DeepSeek raster-group A/B of the CTA-pair FFN (AMOE_GROUP_M / AMOE_GROUP_M_DOWN) + fp32 free-running error
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python tools/fp32_freerun_err.py > gpurun_out/fp32_freerun.jsonl 2>&1
for rep in a b; do
  for gd in 2048 1024 4096 8192; do
    AMOE_GROUP_M_DOWN=$gd timeout 300 python bench.py --config deepseek --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/ds_gmd_${gd}_$rep.json 2>> gpurun_out/ds.err
  done
  for gu in 2048 8192 16384; do
    AMOE_GROUP_M=$gu timeout 300 python bench.py --config deepseek --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/ds_gmu_${gu}_$rep.json 2>> gpurun_out/ds.err
  done
done
cat gpurun_out/fp32_freerun.jsonl; tail -3 gpurun_out/ds.err
for f in gpurun_out/ds_*.json; do python - "$f" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r=d['roofline']
    print(sys.argv[1], round(d['value']), d['clocks']['sm_mhz'], {k: round(v,1) for k,v in r['stage_ms_total'].items() if v}, r['step']['frac_of_schedule_roofline'])
except Exception as e: print(sys.argv[1], 'ERR', e)
PY
done
