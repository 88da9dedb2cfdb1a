#!/bin/bash
# per-CTA timeline of the fused cold kernel on the current code (diagnostic -DAMOE_COLD_TRACE build)
mkdir -p gpurun_out _ab
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
python -m paper_2505_08944_b200.build --out _ab/libamoe_ctrace.so --flags=-DAMOE_COLD_TRACE > gpurun_out/build_ctrace.log 2>&1
for cfg in "deepseek 8 1" "deepseek 8 32" "deepseek 1 1" "deepseek 8 128" "mixtral 1 1" "mixtral 1 128"; do
  set -- $cfg
  AMOE_COLD=1 AMOE_LIB=_ab/libamoe_ctrace.so timeout 120 python tools/cold_trace.py --shape $1 --experts $2 --n $3 2>&1 | tail -1
done | tee gpurun_out/cold_trace_v4.log
timeout 300 python tools/cold_sweep.py --shapes deepseek,mixtral --groups 1,8 --ns 1,16,32,64,128 --modes cold,classic --iters 10 > gpurun_out/cold_sweep_v4.log 2>&1
tail -25 gpurun_out/cold_sweep_v4.log
