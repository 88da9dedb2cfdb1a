#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rf --durations=15 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 2400 bash tools/sanitize.sh
tail -30 gpurun_out/pytest_gpu.log
cat gpurun_out/sanitize_summary.txt
