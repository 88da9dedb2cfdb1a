#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for kk in auto 2,2 1,2 2,4; do
  if [ $kk = auto ]; then unset AMOE_COLD_KAKB; else export AMOE_COLD_KAKB=$kk; fi
  timeout 300 python tools/cold_sweep.py --ns 32,64,128 --modes cold > gpurun_out/cold_kakb_$kk.log 2>&1
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/cold_kakb_*.log')):
    for l in open(f):
        try: r=json.loads(l)
        except: continue
        print(f.split('_')[-1][:-4], r['shape'],r['experts'],r['n'],r['us'],r['frac'])
PY
