cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r34
timeout 900 python tools/ab_env.py batch TIB_CRIT_BATCH_FACTOR=24 TIB_CRIT_BATCH_FACTOR=40 TIB_CRIT_BATCH_FACTOR=64 TIB_CRIT_BATCH_FACTOR=96 > gpurun_out/r34/ab.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -k "batch" > gpurun_out/r34/tests.log 2>&1
