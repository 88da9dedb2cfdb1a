#!/bin/bash
# Algorithm 1 lookahead (W, delta): G-rank emulation (Mixtral G = 2 / 4, DeepSeek G = 4) and the
# N = 1 bench lines, two rounds
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for rep in a b; do
  for cfg in "mixtral 2" "mixtral 4" "deepseek 4"; do
    set -- $cfg; c=$1; G=$2
    for v in "sync 4 0.5" "defrag_global 4 0.5" "defrag_global 8 0.8" "defrag_global 8 0.9" "defrag_global 4 0.8" "defrag_global 8 1.0"; do
      set -- $v
      echo -n "$rep $c G=$G $1 W=$2 delta=$3: "
      timeout 600 python tools/g_emulate.py --config $c --G $G --policy $1 --W $2 --delta $3 --steps 3 2>/dev/null | tail -1 | python -c "import sys,json; r=json.loads(sys.stdin.read()); print(round(r['value']/1e6,3), 'M', 'idle', r.get('idle_frac_per_rank'))"
    done
  done
  for wd in "4 0.5" "8 0.8"; do
    set -- $wd
    echo -n "$rep N=1 mixtral W=$1 delta=$2: "
    timeout 300 python bench.py --W $1 --delta $2 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import sys,json; r=json.loads(sys.stdin.read()); print(round(r['value']/1e6,4), 'M')"
    echo -n "$rep N=1 deepseek W=$1 delta=$2: "
    timeout 300 python bench.py --config deepseek --W $1 --delta $2 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import sys,json; r=json.loads(sys.stdin.read()); print(round(r['value']/1e6,4), 'M')"
  done
done | tee gpurun_out/g_emulate_sweep2.log
