#!/bin/bash
# Round-trip check under gpurun: GPU tests, smoke, and the bench lines (default + variants).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 400 python bench.py > gpurun_out/bench_mixtral.json 2> gpurun_out/bench_mixtral.err
timeout 300 python bench.py --policy sync --no-e2e --no-cpu-baseline > gpurun_out/bench_mixtral_sync.json 2> gpurun_out/bench_mixtral_sync.err
timeout 300 python bench.py --config deepseek --no-cpu-baseline > gpurun_out/bench_deepseek.json 2> gpurun_out/bench_deepseek.err
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
for f in gpurun_out/*.err gpurun_out/*.log; do echo "== $f"; tail -3 $f; done
