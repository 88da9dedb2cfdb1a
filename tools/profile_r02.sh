#!/bin/bash
# Round-2 evidence for profiles/r02 (run under gpurun from the repo root): launch lists of the
# bench commands (time + DRAM bytes per launch), one `ncu --set full` of the pair FFN kernels and
# the combine per shape, and of the fused cold kernel at three cold picks. Summaries are written
# on the box (gpurun copies back <= 64 MiB); the large reports are deleted there.
mkdir -p gpurun_out/p
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/p/build.log 2>&1
K='regex:ffn|combine|gather|drain|enqueue|token_init|announce|splitk|peer_depths|direct_merge'
for cfg in mixtral deepseek; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    -k "$K" --log-file gpurun_out/launches_${cfg}.csv \
    python bench.py --config $cfg --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/p/launches_${cfg}.log 2>&1
  python tools/ncu_summary.py launches gpurun_out/launches_${cfg}.csv > gpurun_out/p/r02_launches_${cfg}.md
  timeout 900 ncu --set full --clock-control none -k regex:"ffn_tc2_kernel|combine_kernel" -s 6 -c 3 \
    -o gpurun_out/full_${cfg} -f \
    python bench.py --config $cfg --steps 1 --warmup 1 --L 2 --no-cpu-baseline --no-e2e > gpurun_out/p/full_${cfg}.log 2>&1
  python tools/ncu_summary.py full gpurun_out/full_${cfg}.ncu-rep > gpurun_out/p/r02_full_${cfg}.md
done
for pc in "mixtral 8 1" "mixtral 1 1" "deepseek 8 16"; do
  set -- $pc
  timeout 600 ncu --set full --clock-control none -k regex:ffn_cold -s 3 -c 1 -o gpurun_out/cold_$1_$2x$3 -f \
    python tools/cold_sweep.py --shapes $1 --groups $2 --ns $3 --modes cold --iters 2 > gpurun_out/p/cold_$1.log 2>&1
  python tools/ncu_summary.py full gpurun_out/cold_$1_$2x$3.ncu-rep > gpurun_out/p/r02_cold_$1_$2x$3.md
done
rm -f gpurun_out/*.ncu-rep gpurun_out/*.csv
du -sh gpurun_out
