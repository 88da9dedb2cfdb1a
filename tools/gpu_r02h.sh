#!/bin/bash
mkdir -p gpurun_out _ab
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
python -m paper_2505_08944_b200.build --out _ab/libamoe_ctrace.so --flags=-DAMOE_COLD_TRACE > gpurun_out/build_ctrace.log 2>&1
for cfg in "deepseek 1 1" "deepseek 8 1" "deepseek 8 64" "mixtral 1 1" "mixtral 8 1"; do
  set -- $cfg
  AMOE_COLD=1 AMOE_LIB=_ab/libamoe_ctrace.so timeout 120 python tools/cold_trace.py --shape $1 --experts $2 --n $3 2>&1 | tail -1
done | tee gpurun_out/cold_trace3.log
