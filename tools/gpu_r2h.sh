cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2h
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r2h/tests.log 2>&1
timeout 300 python bench.py --no-cpu-baseline --steps 3 > gpurun_out/r2h/bench_large.json 2>&1
timeout 400 python bench.py --config batch --no-cpu-baseline --steps 3 > gpurun_out/r2h/bench_batch.json 2>&1
timeout 400 python bench.py --config kronecker --no-cpu-baseline --steps 3 > gpurun_out/r2h/bench_kron.json 2>&1
TIB_CRIT_WORKERS_FACTOR=24 timeout 300 python tools/split_probe.py 2 > gpurun_out/r2h/split2.log 2>&1
