#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_cold.py -q -x -p no:cacheprovider -rf > gpurun_out/pytest_cold.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_cold.log
tail -30 gpurun_out/pytest_cold.log
timeout 900 python tools/cold_sweep.py --out gpurun_out/cold_sweep.json > gpurun_out/cold_sweep.log 2>&1; echo "sweep rc=$?"
tail -60 gpurun_out/cold_sweep.log
