#!/bin/bash
# compute-sanitizer on the final code (tools/sanitize.sh), after a plain run of the same workloads
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python tools/sanitize_run.py all > gpurun_out/sanitize_plain.log 2>&1; echo "plain rc=$?" >> gpurun_out/sanitize_plain.log
cat gpurun_out/sanitize_plain.log
bash tools/sanitize.sh
for f in gpurun_out/sanitize_*.log; do echo "== $f"; grep -E "SUMMARY|token-layers|watchdog|Error|error" $f | tail -4; done
