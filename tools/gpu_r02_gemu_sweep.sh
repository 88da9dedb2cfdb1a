#!/bin/bash
# G-rank emulation: Algorithm 1 lookahead (W, delta) sweep for the box-wide pipelined policy vs sync EP
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for G in 2 4; do
  for v in "sync 4 0.5" "defrag_global 4 0.5" "defrag_global 8 0.5" "defrag_global 16 0.5" "defrag_global 8 0.8" "defrag_global 2 0.5" "defrag_global 0 0.5" "sync 4 0.5"; do
    set -- $v
    echo -n "mixtral G=$G $1 W=$2 delta=$3: "
    timeout 600 python tools/g_emulate.py --config mixtral --G $G --policy $1 --W $2 --delta $3 --steps 3 2>/dev/null | tail -1 | python -c "import sys,json; r=json.loads(sys.stdin.read()); print(round(r['value']/1e6,3), 'M', 'idle', r.get('idle_frac_per_rank'))"
  done
done | tee gpurun_out/g_emulate_sweep.log
