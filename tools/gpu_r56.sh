cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r56
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r56/tests.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/r56/bench_large.json 2>&1
timeout 600 python bench.py --config medium --no-cpu-baseline --steps 5 > gpurun_out/r56/bench_medium.json 2>&1
