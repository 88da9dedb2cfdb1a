#!/bin/bash
# Round-2 state check: build, smoke, every GPU test, the two bench lines, the cold sweep (both modes).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rf --durations=15 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 400 python bench.py > gpurun_out/bench_mixtral.json 2> gpurun_out/bench_mixtral.err
timeout 300 python bench.py --config deepseek --no-cpu-baseline > gpurun_out/bench_deepseek.json 2> gpurun_out/bench_deepseek.err
timeout 900 python tools/cold_sweep.py --ns 1,16,64,128 --out gpurun_out/cold_sweep.json > gpurun_out/cold_sweep.log 2>&1; echo "sweep rc=$?"
tail -5 gpurun_out/smoke.log; tail -25 gpurun_out/pytest_gpu.log
