cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r4
timeout 600 python tools/e2e_timing.py kronecker > gpurun_out/r4/timing_kron.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,smsp__inst_executed.sum --clock-control none -k regex:"rowsum|fill_kernel" -c 4 --csv --log-file gpurun_out/r4/gen.csv python tools/e2e_timing.py large > gpurun_out/r4/ncu_gen.log 2>&1
