cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2y
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2y/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2y/tests.log 2>&1
timeout 300 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/r2y/bench_large.json 2>&1
timeout 300 python bench.py --config medium --no-cpu-baseline --steps 5 > gpurun_out/r2y/bench_medium.json 2>&1
