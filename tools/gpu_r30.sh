cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r30
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r30/tests.log 2>&1
for c in large medium batch kronecker; do
  timeout 400 python bench.py --config $c --no-cpu-baseline --steps 3 > gpurun_out/r30/bench_$c.json 2>&1
done
