#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log; tail -2 gpurun_out/pytest_gpu.log
timeout 400 python bench.py --ungrouped --no-cpu-baseline --no-e2e --steps 2 > gpurun_out/sc_ungr.json 2>&1
timeout 400 python bench.py --config deepseek --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/sc_ds.json 2>&1
timeout 400 python bench.py --config deepseek --T 2048 --no-cpu-baseline --no-e2e --steps 5 > gpurun_out/sc_ds2k.json 2>&1
timeout 400 python bench.py --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/sc_mx.json 2>&1
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/sc_*.json')):
    try:
        r=json.loads(open(f).read().strip().splitlines()[-1]); ro=r['roofline']
        print(f.split('/')[-1], round(r['value']), round(r['ms_per_step'],2), r['clocks']['sm_mhz'], 'busy', r['stall']['busy_frac_rank0'], 'step', ro['step']['frac_of_schedule_roofline'])
    except Exception as e: print(f, 'ERR', e, open(f).read()[-300:])
PY
