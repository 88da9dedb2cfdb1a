#!/bin/bash
# SURVEY.md §8(d) run protocol on the final code: seeds {0,1,2} (median, min/max) for both bench
# shapes, a 20-pass window for Mixtral, a 3-epoch skew-shift run; + the GPU suite
mkdir -p gpurun_out/seeds
S=gpurun_out/seeds
python -c "import __graft_entry__ as g; g.build()" > $S/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $S/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $S/pytest_gpu.log
for seed in 0 1 2; do
  timeout 400 python bench.py --seed $seed --no-cpu-baseline --no-e2e > $S/mixtral_seed$seed.json 2>> $S/err.log
  timeout 400 python bench.py --config deepseek --seed $seed --no-cpu-baseline --no-e2e > $S/deepseek_seed$seed.json 2>> $S/err.log
done
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > $S/mixtral_20pass.json 2>> $S/err.log
timeout 600 python bench.py --steps 6 --warmup 3 --shift-every 64 --no-cpu-baseline --no-e2e > $S/mixtral_shift64.json 2>> $S/err.log
tail -2 $S/pytest_gpu.log
for f in $S/*.json; do python - "$f" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r=d['roofline']
    print(sys.argv[1].split('/')[-1], round(d['value']), d['steps'], d['clocks']['sm_mhz'], d['clocks']['reasons'], round(r['frac'],4), r['step']['frac_of_schedule_roofline'], d['config'].get('skew_epochs_in_timed_region'))
except Exception as e: print(sys.argv[1], 'ERR', e)
PY
done
