#!/bin/bash
# full check after a library change: GPU tests, smoke, bench lines (default, DeepSeek, ungrouped), cold sweep
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rf --durations=5 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 400 python bench.py --no-cpu-baseline > gpurun_out/bench_mixtral.json 2> gpurun_out/bench_mixtral.err
timeout 300 python bench.py --config deepseek --no-cpu-baseline --no-e2e > gpurun_out/bench_deepseek.json 2> gpurun_out/bench_deepseek.err
timeout 400 python bench.py --ungrouped --no-cpu-baseline --no-e2e --steps 2 > gpurun_out/bench_mixtral_ungrouped.json 2> gpurun_out/bench_mixtral_ungrouped.err
tail -3 gpurun_out/smoke.log; tail -12 gpurun_out/pytest_gpu.log
python - <<'PY'
import json
for f in ['bench_mixtral','bench_deepseek','bench_mixtral_ungrouped']:
    try:
        r=json.loads(open(f'gpurun_out/{f}.json').read().strip().splitlines()[-1])
        ro=r['roofline']
        print(f, r['value'], r['ms_per_step'], r['clocks']['sm_mhz'], 'frac', round(ro['frac'],3), 'step', ro.get('step',{}).get('frac_of_schedule_roofline'), 'stages', ro.get('stage_ms_total'))
    except Exception as e: print(f, 'ERR', e)
PY
