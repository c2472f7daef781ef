cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2r
timeout 600 python tools/split_debug.py smoke 3000,200,30,64 mid 4096,300,0,128 > gpurun_out/r2r/debug.log 2>&1
for i in 1 2; do
TIB_SPLIT_STREAMED=1 timeout 300 python bench.py --no-cpu-baseline --steps 3 > gpurun_out/r2r/bench_large_ss$i.json 2>&1
timeout 300 python bench.py --no-cpu-baseline --steps 3 > gpurun_out/r2r/bench_large_nat$i.json 2>&1
done
TIB_SPLIT_STREAMED=1 timeout 300 python bench.py --config medium --no-cpu-baseline --steps 3 > gpurun_out/r2r/bench_medium_ss.json 2>&1
