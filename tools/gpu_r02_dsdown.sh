#!/bin/bash
# one DeepSeek down-GEMM launch (bench shape) under ncu --set full with source counters; the
# report comes back for `ncu -i --page source` analysis
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"ffn_tc2_kernel" -s 4 -c 2 \
  -o gpurun_out/ds_ffn -f python bench.py --config deepseek --steps 1 --warmup 1 --L 2 --no-cpu-baseline --no-e2e > gpurun_out/ds_ffn.log 2>&1
ls -la gpurun_out
