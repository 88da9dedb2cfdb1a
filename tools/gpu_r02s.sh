#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for cfg in "mixtral 2" "mixtral 4" "deepseek 4"; do
  set -- $cfg; c=$1; G=$2
  echo -n "$c G=$G global_heur: "
  AMOE_PIPELINE=0 timeout 600 python tools/g_emulate.py --config $c --G $G --policy defrag_global --steps 3 2>/dev/null | tail -1 | python -c "import sys,json; r=json.loads(sys.stdin.read()); print(round(r['value']/1e6,3), 'M', 'idle', r.get('idle_frac_per_rank'))"
done | tee gpurun_out/g_emulate_r02b.log
# small-T waves: cold picks inside the real loop
for T in 512 2048; do
  for cold in auto 0; do
    if [ $cold = auto ]; then unset AMOE_COLD; else export AMOE_COLD=0; fi
    timeout 300 python bench.py --config deepseek --T $T --no-cpu-baseline --no-e2e --steps 5 > gpurun_out/smallT_ds_${T}_$cold.json 2>&1
    timeout 300 python bench.py --config mixtral --T $T --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/smallT_mx_${T}_$cold.json 2>&1
  done
done
unset AMOE_COLD
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/smallT_*.json')):
    try:
        r=json.loads(open(f).read().strip().splitlines()[-1]); ro=r['roofline']
        print(f.split('/')[-1], round(r['value']), round(r['ms_per_step'],2), r['clocks']['sm_mhz'], 'step', ro['step']['frac_of_schedule_roofline'], 'cold', ro['stage_ms_total'].get('ffn_cold'), ro['stage_launches'].get('ffn_cold'), 'gu', ro['stage_ms_total']['ffn_gateup'])
    except Exception as e: print(f, 'ERR', e, open(f).read()[-300:])
PY
