#!/bin/bash
# One GPU call's worth of evidence for profiles/ (run under gpurun from the repo root):
# launch lists of the bench command (cold-cache, serialised: compare shares) and one
# `ncu --set full` capture of the FFN pair kernels per configuration.
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for cfg in mixtral deepseek; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${cfg}.csv \
    python bench.py --config $cfg --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/launches_${cfg}.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:ffn_tc2_kernel -s 4 -c 2 \
    -o gpurun_out/ffn_full_${cfg} -f \
    python bench.py --config $cfg --steps 1 --warmup 1 --L 2 --no-cpu-baseline --no-e2e > gpurun_out/ffn_full_${cfg}.log 2>&1
done
ls -la gpurun_out
