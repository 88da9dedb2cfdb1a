#!/bin/bash
# fused cold kernel: per-slice activation dependencies (in-tree) vs the previous whole-queue
# dependency (_ab/libamoe_head.so), alternating; + the cold GPU tests on the new build
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_cold.py tests/test_gpu_replay.py -x -q > gpurun_out/pytest_cold.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_cold.log
for rep in a b; do
  for lib in new head; do
    if [ $lib = head ]; then export AMOE_LIB=_ab/libamoe_head.so; else unset AMOE_LIB; fi
    timeout 300 python tools/cold_sweep.py --shapes deepseek,mixtral --groups 1,8 --ns 1,16,32,64,128 --modes cold --iters 10 > gpurun_out/slice_${lib}_$rep.log 2>&1
  done
done
unset AMOE_LIB
tail -2 gpurun_out/pytest_cold.log
python - <<'PY'
import json,glob
t={}
for f in sorted(glob.glob('gpurun_out/slice_*.log')):
    lib=f.split('_')[1]
    for l in open(f):
        try: r=json.loads(l)
        except: continue
        t.setdefault((r['shape'],r['experts'],r['n']),{}).setdefault(lib,[]).append((r['us'], r['frac']))
for k,v in sorted(t.items()): print(*k, {p: [x for x in u] for p,u in sorted(v.items())})
PY
