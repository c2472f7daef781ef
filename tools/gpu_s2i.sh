cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/s2i
TIB_LIB_VARIANT=prof TIB_CHAIN_PROF=1 timeout 300 python tools/prof_run.py large 1 > gpurun_out/s2i/chainprof.log 2>&1
TIB_LIB_VARIANT=prof2 TIB_CHAIN_PROF=1 timeout 300 python tools/prof_run.py large 1 > gpurun_out/s2i/chainprof_f2.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s2i/bench.json 2> gpurun_out/s2i/bench.err
TIB_LIB_VARIANT=f2 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s2i/bench_f2.json 2> gpurun_out/s2i/bench_f2.err
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_configs.py -m gpu -x -q -p no:cacheprovider > gpurun_out/s2i/gpu_tests.log 2>&1
