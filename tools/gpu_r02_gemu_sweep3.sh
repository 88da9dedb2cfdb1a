#!/bin/bash
# Mixtral G = 2 / 4: sync EP vs the box-wide pipelined Algorithm 1 at W in {8, 12, 16}, δ = 1.0 (3 rounds)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for rep in a b c; do
  for G in 2 4; do
    for v in "sync 4 0.5" "defrag_global 8 1.0" "defrag_global 12 1.0" "defrag_global 16 1.0"; do
      set -- $v
      echo -n "$rep mixtral G=$G $1 W=$2 delta=$3: "
      timeout 600 python tools/g_emulate.py --config mixtral --G $G --policy $1 --W $2 --delta $3 --steps 3 2>/dev/null | tail -1 | python -c "import sys,json; r=json.loads(sys.stdin.read()); print(round(r['value']/1e6,3), 'M')"
    done
  done
done | tee gpurun_out/g_emulate_sweep3.log
