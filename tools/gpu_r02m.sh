#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:ffn_cold -s 3 -c 1 -o gpurun_out/cold_mx1x128 -f \
  python tools/cold_sweep.py --shapes mixtral --groups 1 --ns 128 --modes cold --iters 2 > gpurun_out/ncu_mx.log 2>&1; echo "ncu rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:ffn_cold -s 3 -c 1 -o gpurun_out/cold_mx1x1 -f \
  python tools/cold_sweep.py --shapes mixtral --groups 1 --ns 1 --modes cold --iters 2 > gpurun_out/ncu_mx1.log 2>&1; echo "ncu rc=$?"
