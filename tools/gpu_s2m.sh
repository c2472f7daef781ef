cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/s2m
for sh in 0 2 4; do
  TIB_POLL_SHIFT=$sh timeout 300 python tools/e2e_timing.py batch > gpurun_out/s2m/batch_$sh.log 2>&1
  TIB_POLL_SHIFT=$sh timeout 300 python tools/e2e_probe.py large > gpurun_out/s2m/large_$sh.log 2>&1
done
