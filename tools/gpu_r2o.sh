cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2o
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "two_chain or streamed" > gpurun_out/r2o/tests.log 2>&1
timeout 300 python bench.py --no-cpu-baseline --steps 3 > gpurun_out/r2o/bench_large.json 2>&1
TIB_SPLIT_AGENTS=8 timeout 300 python bench.py --no-cpu-baseline --steps 3 > gpurun_out/r2o/bench_large_a8.json 2>&1
TIB_SPLIT=0 timeout 300 python bench.py --no-cpu-baseline --steps 3 > gpurun_out/r2o/bench_large_nat.json 2>&1
TIB_HOST_TIMING=1 timeout 300 python tools/e2e_timing.py large > gpurun_out/r2o/e2e_large.log 2>&1
