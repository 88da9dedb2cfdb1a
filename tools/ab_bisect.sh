# A/B of FFN microbenchmark across builds in _ab/* (scratch worktrees), interleaved
R=$GRAFT_REPO_ROOT
run() { (cd $1 && env $2 timeout 120 python tools/ffn_micro.py --variants ${V:-2cta:2048} --secs 4 2>&1 | grep variant | sed "s|^|$(basename $1) $2 |"); }
for i in 1 2; do
  for d in $DIRS; do run $R/$d ""; done
done
