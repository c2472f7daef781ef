# round-2 profiles of the current build: bench launch list (large), ncu --set full of both sweeps
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/prof
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/prof/launches_bench.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/prof/bench_under_ncu.log 2>&1
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:dataflow_kernel -c 2 \
    -o gpurun_out/prof/large_sweeps python tools/prof_run.py large 1 > gpurun_out/prof/ncu_full.log 2>&1
