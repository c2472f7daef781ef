cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r42
export TIB_WATCHDOG_S=5
TIB_SPLIT_AGENTS=1 timeout 900 python tools/stress_split.py 100000,1000,100,256 150 > gpurun_out/r42/a1.log 2>&1
TIB_SPLIT_AGENTS=2 timeout 900 python tools/stress_split.py 100000,1000,100,256 100 > gpurun_out/r42/a2.log 2>&1
unset TIB_WATCHDOG_S
for a in 1 2 8; do TIB_SPLIT_AGENTS=$a timeout 300 python bench.py --config medium --no-cpu-baseline --steps 3 > gpurun_out/r42/bench_medium_a$a.json 2>&1; done
