#!/bin/bash
# Final round-2 evidence on one B200 (after the launch-count reductions): build, smoke, the GPU suite, the bench lines (Mixtral with
# cpu_baseline + e2e, DeepSeek, the reference arm), then ncu launch lists + `--set full` captures
# (summaries only) into gpurun_out/final2/.
mkdir -p gpurun_out/final2
F=gpurun_out/final2
python -c "import __graft_entry__ as g; g.build()" > $F/build.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $F/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $F/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $F/pytest_gpu.log
timeout 600 python bench.py > $F/bench_mixtral.json 2> $F/bench_mixtral.err
timeout 400 python bench.py --config deepseek > $F/bench_deepseek.json 2> $F/bench_deepseek.err
timeout 400 python bench.py --impl reference --steps 2 --warmup 3 > $F/bench_reference.json 2> $F/bench_reference.err
for rep in a b; do
  for ev in 0 1; do
    AMOE_BENCH_STAGE_EVENTS=$ev timeout 300 python bench.py --no-cpu-baseline --no-e2e > $F/ev${ev}_mixtral_$rep.json 2>> $F/ev.err
    AMOE_BENCH_STAGE_EVENTS=$ev timeout 300 python bench.py --config deepseek --no-cpu-baseline --no-e2e > $F/ev${ev}_deepseek_$rep.json 2>> $F/ev.err
  done
done
K='regex:ffn|combine|gather|drain|enqueue|token_init|announce|splitk|peer_depths|direct_merge'
for cfg in mixtral deepseek; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    -k "$K" --log-file gpurun_out/launches_${cfg}.csv \
    python bench.py --config $cfg --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $F/launches_${cfg}.log 2>&1
  python tools/ncu_summary.py launches gpurun_out/launches_${cfg}.csv > $F/launches_${cfg}.md
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"ffn_tc2_kernel|combine_kernel|gather_kernel" -s 8 -c 4 \
    -o gpurun_out/full_${cfg} -f \
    python bench.py --config $cfg --steps 1 --warmup 1 --L 2 --no-cpu-baseline --no-e2e > $F/full_${cfg}.log 2>&1
  python tools/ncu_summary.py full gpurun_out/full_${cfg}.ncu-rep > $F/full_${cfg}.md
done
for pc in "mixtral 8 1" "mixtral 1 1" "deepseek 8 16"; do
  set -- $pc
  timeout 600 ncu --set full --clock-control none -k regex:ffn_cold -s 3 -c 1 -o gpurun_out/cold_$1_$2x$3 -f \
    python tools/cold_sweep.py --shapes $1 --groups $2 --ns $3 --modes cold --iters 2 > $F/cold_$1.log 2>&1
  python tools/ncu_summary.py full gpurun_out/cold_$1_$2x$3.ncu-rep > $F/cold_$1_$2x$3.md
done
rm -f gpurun_out/*.ncu-rep gpurun_out/*.csv
tail -3 $F/pytest_gpu.log; tail -2 $F/smoke.log
for f in $F/bench_*.json $F/ev*.json; do python - "$f" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    r=d.get('roofline',{})
    print(sys.argv[1], round(d.get('value',0)), d.get('e2e',{}).get('value'), d.get('clocks',{}).get('sm_mhz'), r.get('frac'), {k:v.get('frac') for k,v in r.get('hbm_kernels',{}).items()}, r.get('step',{}).get('frac_of_schedule_roofline'))
except Exception as e: print(sys.argv[1], 'ERR', e)
PY
done
du -sh gpurun_out
