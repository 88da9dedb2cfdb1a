#!/bin/bash
# A/B of the in-tree build against _ab/libamoe_base.so on bench lines (interleaved, two rounds)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
ARGS=${ARGS:---no-cpu-baseline --no-e2e --steps 3}
for round in 1 2; do
for cfgname in mixtral deepseek; do
  for lib in base new; do
    if [ $lib = base ]; then export AMOE_LIB=_ab/libamoe_base.so; else unset AMOE_LIB; fi
    timeout 400 python bench.py --config $cfgname $ARGS > gpurun_out/ab_${cfgname}_${lib}_$round.json 2> gpurun_out/ab_${cfgname}_${lib}_$round.err
  done
done
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/ab_*.json')):
    try:
        r=json.loads(open(f).read().strip().splitlines()[-1]); ro=r['roofline']
        print(f.split('/')[-1], round(r['value']), r['clocks']['sm_mhz'], 'combine', ro['stage_ms_total']['combine'], ro['hbm_kernels'].get('combine',{}).get('frac'), 'rebatch', ro['stage_ms_total']['rebatch'], 'gu', ro['stage_ms_total']['ffn_gateup'])
    except Exception as e: print(f, 'ERR', e)
PY
