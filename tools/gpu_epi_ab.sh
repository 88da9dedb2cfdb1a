#!/bin/bash
# Epilogue merge A/B (AMOE_EPI_MERGE=0 / 1): the new tests, then bench stage times, alternating
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_epi_merge.py -x -q > gpurun_out/pytest_epi.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_epi.log
for rep in a b; do
  for em in 0 1; do
    AMOE_EPI_MERGE=$em timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/epi_mixtral_${em}_$rep.json 2>> gpurun_out/epi_bench.err
    AMOE_EPI_MERGE=$em timeout 300 python bench.py --config deepseek --no-cpu-baseline --no-e2e > gpurun_out/epi_deepseek_${em}_$rep.json 2>> gpurun_out/epi_bench.err
  done
done
tail -3 gpurun_out/pytest_epi.log; tail -3 gpurun_out/epi_bench.err
for f in gpurun_out/epi_*.json; do python - "$f" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r=d['roofline']
    print(sys.argv[1], round(d['value']), d['clocks']['sm_mhz'], {k: round(v,1) for k,v in r['stage_ms_total'].items()}, r['step']['frac_of_schedule_roofline'])
except Exception as e: print(sys.argv[1], 'ERR', e)
PY
done
