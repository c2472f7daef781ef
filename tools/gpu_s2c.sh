# signal agent: chain profile, trace, parity tests, bench (and TIB_AGENT=0 for comparison)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/s2c
TIB_LIB_VARIANT=prof TIB_CHAIN_PROF=1 timeout 300 python tools/prof_run.py large 1 > gpurun_out/s2c/chainprof_large.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/s2c/gpu_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/s2c/gpu_tests.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s2c/bench.json 2> gpurun_out/s2c/bench.err
TIB_AGENT=0 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s2c/bench_noagent.json 2> gpurun_out/s2c/bench_noagent.err
bash tools/trace_run.sh large > gpurun_out/s2c/trace_run.log 2>&1
cp gpurun_out/tr/report_large.txt gpurun_out/s2c/ 2>/dev/null
