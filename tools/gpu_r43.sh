cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r43
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r43/tests.log 2>&1
timeout 300 python bench.py --config medium --no-cpu-baseline --steps 3 > gpurun_out/r43/bench_medium.json 2>&1
timeout 300 python bench.py --no-cpu-baseline --steps 3 > gpurun_out/r43/bench_large.json 2>&1
export TIB_WATCHDOG_S=5
timeout 900 python tools/stress_split.py 100000,1000,100,256 60 > gpurun_out/r43/stress_medium.log 2>&1
timeout 900 python tools/stress_split.py 200000,2000,200,512 20 > gpurun_out/r43/stress_large.log 2>&1
