#!/bin/bash
# G-rank emulation on one GPU on the final code: sync EP vs asynchronous policies
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
run() {  # name, env..., args
  local name=$1; shift
  env "$@" > /dev/null
}
for cfg in "mixtral 2" "mixtral 4" "deepseek 4" "mixtral 8"; do
  set -- $cfg; c=$1; G=$2
  for v in sync defrag defrag_heur defrag_pipe global_pipe; do
    case $v in
      sync) E="" ; P=sync ;;
      defrag) E="" ; P=defrag ;;
      defrag_heur) E="AMOE_PIPELINE=0" ; P=defrag ;;
      defrag_pipe) E="AMOE_GROW_WAIT=0 AMOE_COMBINE_FIRST=0" ; P=defrag ;;
      global_pipe) E="AMOE_GROW_WAIT=0 AMOE_COMBINE_FIRST=0" ; P=defrag_global ;;
    esac
    echo -n "$c G=$G $v: "
    env $E timeout 600 python tools/g_emulate.py --config $c --G $G --policy $P --steps 3 2>/dev/null | tail -1 | python -c "import sys,json; r=json.loads(sys.stdin.read()); print(round(r['value']/1e6,3), 'M', 'idle', r.get('idle_frac_per_rank'), 'execs', r.get('executions', r.get('picks')))"
  done
done | tee gpurun_out/g_emulate_final.log
