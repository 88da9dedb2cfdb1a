#!/bin/bash
# pair (M=256) vs 1-CTA (M=128) FFN kernels on the four-kernel path around the n = 257..511 cliff
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for one in 0 1; do
  AMOE_FFN_1CTA=$one timeout 900 python tools/cold_sweep.py --shapes mixtral,deepseek --groups 1,8 \
    --ns 192,256,320,384,448,512,640,768,1024,1536 --modes classic --iters 10 > gpurun_out/m128_$one.log 2>&1
done
for one in 1 0; do
  AMOE_FFN_1CTA=$one timeout 400 python bench.py --config deepseek --no-cpu-baseline --no-e2e > gpurun_out/m128_bench_ds_$one.json 2>&1
done
python - <<'PY'
import json
t={}
for one in (0,1):
    for l in open(f'gpurun_out/m128_{one}.log'):
        try: r=json.loads(l)
        except: continue
        t.setdefault((r['shape'],r['experts'],r['n']),{})[one]=r['us']
for k,v in t.items(): print(*k, 'pair', v.get(0), '1cta', v.get(1))
for one in (1,0):
    d=json.loads(open(f'gpurun_out/m128_bench_ds_{one}.json').read().strip().splitlines()[-1])
    print('deepseek bench 1cta=%d'%one, round(d['value']), d['roofline']['stage_ms_total'])
PY
