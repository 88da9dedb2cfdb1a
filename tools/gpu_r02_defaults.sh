#!/bin/bash
# new G > 1 defaults (pipelined loop; bench policy defrag_global): GPU suite, N = 1 bench lines,
# the N = 2 bench path with two ranks sharing the GPU (gloo), and the reference arm under torchrun
mkdir -p gpurun_out/defaults
D=gpurun_out/defaults
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $D/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $D/pytest_gpu.log
timeout 400 python bench.py --no-cpu-baseline > $D/bench_mixtral.json 2> $D/bench_mixtral.err
timeout 400 python bench.py --config deepseek --no-cpu-baseline --no-e2e > $D/bench_deepseek.json 2> $D/bench_deepseek.err
AMOE_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --T 4096 --no-cpu-baseline > $D/bench_n2.json 2> $D/bench_n2.err
AMOE_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29534 bench.py --impl reference --gpus 2 --steps 1 --warmup 3 > $D/bench_ref_n2.json 2> $D/bench_ref_n2.err
tail -3 $D/pytest_gpu.log
for f in $D/bench_*.json; do echo "== $f"; tail -c 700 $f; echo; done
tail -3 $D/bench_n2.err
