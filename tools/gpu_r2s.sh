cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2s
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_configs.py -q -x -p no:cacheprovider > gpurun_out/r2s/tests.log 2>&1
timeout 300 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/r2s/bench_large.json 2>&1
timeout 300 python bench.py --config medium --no-cpu-baseline --steps 5 > gpurun_out/r2s/bench_medium.json 2>&1
