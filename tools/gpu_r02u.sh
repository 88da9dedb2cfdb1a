#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for round in 1 2; do
for v in 0 1; do
  AMOE_DOWN_1CTA=$v timeout 400 python bench.py --config deepseek --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/d1_ds_${v}_$round.json 2>&1
done
done
AMOE_DOWN_1CTA=1 timeout 400 python bench.py --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/d1_mx_1.json 2>&1
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/d1_*.json')):
    try:
        r=json.loads(open(f).read().strip().splitlines()[-1]); ro=r['roofline']
        print(f.split('/')[-1], round(r['value']), round(r['ms_per_step'],2), r['clocks']['sm_mhz'], 'gu', ro['stage_ms_total']['ffn_gateup'], 'down', ro['stage_ms_total']['ffn_down'], 'down TF', round(ro['down_kernel_tflops']))
    except Exception as e: print(f, 'ERR', e, open(f).read()[-300:])
PY
