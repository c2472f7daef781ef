cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/s2n
for p in 0 8 16 32; do
  TIB_BATCH_PIPE=$p timeout 300 python tools/e2e_timing.py batch > gpurun_out/s2n/batch_$p.log 2>&1
done
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "batch" > gpurun_out/s2n/tests.log 2>&1
