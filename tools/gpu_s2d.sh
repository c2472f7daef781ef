# sweep interference microbenchmarks + chain profile / bench with the two-column lookahead
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/s2d
for m in 0 1 2; do timeout 60 tools/bin/sweep_bench_f$m > gpurun_out/s2d/sweep_f$m.log 2>&1; done
TIB_LIB_VARIANT=prof TIB_CHAIN_PROF=1 timeout 300 python tools/prof_run.py large 1 > gpurun_out/s2d/chainprof_large.log 2>&1
TIB_AGENT=0 TIB_LIB_VARIANT=prof TIB_CHAIN_PROF=1 timeout 300 python tools/prof_run.py large 1 > gpurun_out/s2d/chainprof_large_noagent.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s2d/bench.json 2> gpurun_out/s2d/bench.err
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider > gpurun_out/s2d/gpu_tests.log 2>&1
