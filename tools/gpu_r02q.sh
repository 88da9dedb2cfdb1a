#!/bin/bash
# pipelined scheduler: all GPU tests, then bench A/B pipeline on/off
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
#timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
#
for pl in 1 0; do
  AMOE_PIPELINE=$pl timeout 400 python bench.py --ungrouped --no-cpu-baseline --no-e2e --steps 2 > gpurun_out/pl_ungrouped_$pl.json 2>&1
  AMOE_PIPELINE=$pl timeout 400 python bench.py --config deepseek --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/pl_deepseek_$pl.json 2>&1
  AMOE_PIPELINE=$pl timeout 400 python bench.py --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/pl_mixtral_$pl.json 2>&1
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/pl_*.json')):
    try:
        r=json.loads(open(f).read().strip().splitlines()[-1]); ro=r['roofline']
        print(f.split('/')[-1], round(r['value']), round(r['ms_per_step'],1), r['clocks']['sm_mhz'], 'step', ro['step']['frac_of_schedule_roofline'], 'busy', r['stall']['busy_frac_rank0'])
    except Exception as e: print(f, 'ERR', e, open(f).read()[-400:])
PY
