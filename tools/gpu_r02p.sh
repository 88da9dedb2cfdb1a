#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_direct.py -q -p no:cacheprovider -rf > gpurun_out/pytest_p.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_p.log
tail -3 gpurun_out/pytest_p.log
timeout 300 python bench.py --no-cpu-baseline --no-e2e --shift-every 32 > gpurun_out/bench_shift.json 2> gpurun_out/bench_shift.err
timeout 300 python bench.py --no-cpu-baseline --no-e2e --topk 1 > gpurun_out/bench_top1.json 2> gpurun_out/bench_top1.err
timeout 300 python bench.py --no-cpu-baseline --no-e2e --topk 1 --direct > gpurun_out/bench_top1_direct.json 2> gpurun_out/bench_top1_direct.err
timeout 400 python bench.py --ungrouped --no-cpu-baseline --no-e2e --steps 2 > gpurun_out/bench_mixtral_ungrouped.json 2> gpurun_out/bench_mixtral_ungrouped.err
AMOE_DIST_BACKEND=gloo timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 3 --T 4096 --no-e2e > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err
python - <<'PY'
import json
for f in ['bench_shift','bench_top1','bench_top1_direct','bench_mixtral_ungrouped','bench_n2']:
    try:
        r=json.loads(open(f'gpurun_out/{f}.json').read().strip().splitlines()[-1])
        ro=r['roofline']
        print(f, round(r['value']), round(r['ms_per_step'],1), r['clocks']['sm_mhz'], 'step', ro['step']['frac_of_schedule_roofline'], 'nv', json.dumps(ro.get('nvlink'))[:300], r.get('placement'), r.get('skew_epochs_in_timed_region'), 'stages', ro['stage_ms_total'])
    except Exception as e: print(f, 'ERR', e, open(f'gpurun_out/{f}.err').read()[-500:])
PY
