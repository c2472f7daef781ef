cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2c
timeout 900 python tools/crit_sweep.py large 56,12 0,12 8,12 16,12 24,12 40,12 56,0 56,4 56,24 > gpurun_out/r2c/crit_large.log 2>&1
timeout 900 python tools/crit_sweep.py batch 56,12 0,0 8,4 24,8 96,24 > gpurun_out/r2c/crit_batch.log 2>&1
TIB_HOST_TIMING=1 timeout 300 python tools/e2e_timing.py large > gpurun_out/r2c/e2e_large.log 2>&1
