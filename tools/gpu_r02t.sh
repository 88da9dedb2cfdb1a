#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for T in 512 2048 4096; do
  for ms in 1 0; do
    AMOE_MIXED_SPLIT=$ms timeout 300 python bench.py --config deepseek --T $T --no-cpu-baseline --no-e2e --steps 5 > gpurun_out/mix_ds_${T}_$ms.json 2>&1
  done
done
for ms in 1 0; do
  AMOE_MIXED_SPLIT=$ms timeout 400 python bench.py --config deepseek --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/mix_ds_16384_$ms.json 2>&1
  AMOE_MIXED_SPLIT=$ms timeout 400 python bench.py --ungrouped --no-cpu-baseline --no-e2e --steps 2 > gpurun_out/mix_mx_ungr_$ms.json 2>&1
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/mix_*.json')):
    try:
        r=json.loads(open(f).read().strip().splitlines()[-1]); ro=r['roofline']
        print(f.split('/')[-1], round(r['value']), round(r['ms_per_step'],2), r['clocks']['sm_mhz'], 'step', ro['step']['frac_of_schedule_roofline'], 'cold', ro['stage_ms_total'].get('ffn_cold'), ro['stage_launches'].get('ffn_cold'), 'gu', ro['stage_ms_total']['ffn_gateup'])
    except Exception as e: print(f, 'ERR', e, open(f).read()[-300:])
PY
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "parity or cold or direct or replay" 2>&1 | tail -2
