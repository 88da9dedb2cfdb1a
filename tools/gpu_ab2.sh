#!/bin/bash
# A/B of two builds in one call: $AB_BASE (AMOE_LIB) vs the in-tree build; parity tests of the in-tree build first
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_direct.py -q -x -p no:cacheprovider > gpurun_out/pytest_ab.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ab.log
tail -2 gpurun_out/pytest_ab.log
BASE=${AB_BASE:-paper_2505_08944_b200/lib/ab/libamoe_base.so}
for cfg in ${AB_CFGS:-deepseek mixtral}; do
  for v in new base new base; do
    if [ $v = base ]; then export AMOE_LIB=$PWD/$BASE; else unset AMOE_LIB; fi
    timeout 400 python bench.py --config $cfg --no-cpu-baseline --no-e2e > gpurun_out/ab2_${cfg}_$v.json 2> gpurun_out/ab2_${cfg}_$v.err
    python - <<PY
import json
d=json.loads(open('gpurun_out/ab2_${cfg}_${v}.json').read().strip().splitlines()[-1])
r=d['roofline']
print('${cfg}', '${v}', round(d['value']), 'gu', round(r['frac'],4), 'comb', r['hbm_kernels']['combine']['frac'], r['stage_ms_total'], 'clk', d['clocks']['sm_mhz'], 'step', r['step']['frac_of_schedule_roofline'])
PY
  done
done
unset AMOE_LIB
