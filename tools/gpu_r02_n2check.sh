#!/bin/bash
# bench.py with the final defaults: N = 1 (Mixtral) and the N = 2 path with two ranks sharing the GPU
mkdir -p gpurun_out/n2check
D=gpurun_out/n2check
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
timeout 400 python bench.py --no-cpu-baseline --no-e2e > $D/bench_mixtral_n1.json 2> $D/n1.err
AMOE_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29535 bench.py --gpus 2 --steps 3 --warmup 3 --T 4096 --no-cpu-baseline > $D/bench_n2.json 2> $D/n2.err
for f in $D/*.json; do python - "$f" <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], round(d['value']), d['n_gpus'], d['config']['policy'], d['config']['lookahead'], d['stall']['idle_frac_per_rank'])
PY
done
tail -2 $D/n2.err
