#!/bin/bash
# ncu --set full of the gate/up pair kernel with the cp.async gather (source-level stalls)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:ffn_tc2 -s 2 -c 1 -o gpurun_out/cpg -f \
  python bench.py --config mixtral --steps 1 --warmup 1 --L 2 --no-cpu-baseline --no-e2e > gpurun_out/cpg.log 2>&1
ncu -i gpurun_out/cpg.ncu-rep --page details > gpurun_out/cpg_details.txt 2>&1
ncu -i gpurun_out/cpg.ncu-rep --page source --csv > gpurun_out/cpg_source.csv 2>&1
ncu -i gpurun_out/cpg.ncu-rep --page raw --csv > gpurun_out/cpg_raw.csv 2>&1
rm -f gpurun_out/cpg.ncu-rep
ls -la gpurun_out
