#!/bin/bash
# ncu source-level capture of the combine kernel (DeepSeek layer), base build and in-tree build
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for v in base new; do
  if [ $v = base ]; then export AMOE_LIB=$PWD/paper_2505_08944_b200/lib/ab/libamoe_base.so; else unset AMOE_LIB; fi
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:combine_kernel -s 6 -c 1 -o gpurun_out/comb_$v -f \
    python bench.py --config deepseek --steps 1 --warmup 1 --L 4 --no-cpu-baseline --no-e2e > gpurun_out/comb_$v.log 2>&1
  ncu -i gpurun_out/comb_$v.ncu-rep --page details > gpurun_out/comb_${v}_details.txt 2>&1
  ncu -i gpurun_out/comb_$v.ncu-rep --page source --csv > gpurun_out/comb_${v}_source.csv 2>&1
  ncu -i gpurun_out/comb_$v.ncu-rep --page raw --csv > gpurun_out/comb_${v}_raw.csv 2>&1
  rm -f gpurun_out/comb_$v.ncu-rep
done
