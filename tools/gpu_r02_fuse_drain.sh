#!/bin/bash
# host-decided drain inside the gather + combine-ring snapshot inside the combine (G = 1): GPU suite + bench A/B vs the previous build
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
for rep in a b; do
  for lib in new head; do
    if [ $lib = new ]; then unset AMOE_LIB; else export AMOE_LIB=_ab/libamoe_prev.so; fi
    timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/fe_mixtral_${lib}_$rep.json 2>> gpurun_out/nr.err
    timeout 300 python bench.py --config deepseek --no-cpu-baseline --no-e2e > gpurun_out/fe_deepseek_${lib}_$rep.json 2>> gpurun_out/nr.err
    timeout 300 python bench.py --ungrouped --steps 3 --no-cpu-baseline --no-e2e > gpurun_out/fe_ungrouped_${lib}_$rep.json 2>> gpurun_out/nr.err
  done
done
unset AMOE_LIB
tail -2 gpurun_out/pytest_gpu.log
for f in gpurun_out/fe_*.json; do python - "$f" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r=d['roofline']
    print(sys.argv[1].split('/')[-1], round(d['value']), d['gpu_launches'], d['clocks']['sm_mhz'], r['step']['frac_of_schedule_roofline'], d['stall']['busy_frac_rank0'], r['stage_ms_total']['rebatch'], r['hbm_kernels'].get('rebatch',{}).get('frac'))
except Exception as e: print(sys.argv[1], 'ERR', e)
PY
done
