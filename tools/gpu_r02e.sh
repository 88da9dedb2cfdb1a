#!/bin/bash
# cold-path measurement: device-only sweep + ncu launch list and one full capture of the fused cold kernel
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python tools/cold_sweep.py --ns 1,16,64,128 --out gpurun_out/cold_sweep2.json > gpurun_out/cold_sweep2.log 2>&1; echo "sweep rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/cold_launches.csv python tools/cold_sweep.py --shapes deepseek,mixtral --groups 1,8 --ns 1,64,128 --iters 3 > gpurun_out/cold_ncu_run.log 2>&1; echo "ncu rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:ffn_cold -s 2 -c 1 -o gpurun_out/cold_ds8x64 -f \
  python tools/cold_sweep.py --shapes deepseek --groups 8 --ns 64 --modes cold --iters 2 > gpurun_out/cold_full.log 2>&1; echo "ncu full rc=$?"
python - <<'PY'
import json
for l in open('gpurun_out/cold_sweep2.log'):
    try: r=json.loads(l)
    except: continue
    print(r['shape'],r['experts'],r['n'],r['mode'],r['us'],r['frac'])
PY
