cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r35
for p in 16 8 32; do
  TIB_BATCH_PIPE=$p timeout 300 python tools/e2e_timing.py batch > gpurun_out/r35/batch_$p.log 2>&1
done
