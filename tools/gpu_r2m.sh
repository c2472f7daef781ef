cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2m
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2m/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2m/tests.log 2>&1
timeout 300 python bench.py --no-cpu-baseline --steps 3 > gpurun_out/r2m/bench_large.json 2>&1
timeout 300 python bench.py --config medium --no-cpu-baseline --steps 3 > gpurun_out/r2m/bench_medium.json 2>&1
TIB_SPLIT=0 timeout 300 python bench.py --config medium --no-cpu-baseline --steps 3 > gpurun_out/r2m/bench_medium_nat.json 2>&1
