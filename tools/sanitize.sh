#!/bin/bash
# compute-sanitizer over the tiny config and loopback G=2 (run under gpurun from the repo root);
# logs go to gpurun_out/sanitize_*.log (summaries copied to profiles/ by hand).
mkdir -p gpurun_out
export AMOE_DIE_PROBE=0
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck racecheck; do
  for what in single loopback cold direct global; do
    timeout 900 $CS --tool $tool --print-limit 50 --error-exitcode 9 \
      python tools/sanitize_run.py $what > gpurun_out/sanitize_${tool}_${what}.log 2>&1
    echo "$tool $what rc=$?" | tee -a gpurun_out/sanitize_summary.txt
  done
done
