#!/bin/bash
# cp.async gather fused into the gate/up producer: parity tests + A/B bench (materialised gather vs fused)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -p no:cacheprovider > gpurun_out/pytest_full.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_full.log
tail -3 gpurun_out/pytest_full.log
for cfg in mixtral deepseek; do
  for cg in 1 0 1; do
    AMOE_CP_GATHER=$cg timeout 400 python bench.py --config $cfg --no-cpu-baseline --no-e2e > gpurun_out/ab_${cfg}_${cg}.json 2> gpurun_out/ab_${cfg}_${cg}.err
    python - <<PY
import json
d=json.loads(open('gpurun_out/ab_${cfg}_${cg}.json').read().strip().splitlines()[-1])
r=d['roofline']
print('${cfg}', 'cp=${cg}', round(d['value']), 'gu', round(r['frac'],4), 'stage', r['stage_ms_total'], 'clk', d['clocks']['sm_mhz'], 'step', r['step']['frac_of_schedule_roofline'])
PY
  done
done
