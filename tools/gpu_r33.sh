cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r33
timeout 900 python tools/ab_env.py batch TIB_BATCH_CHAIN=0 TIB_BATCH_CHAIN=1 TIB_BATCH_CHAIN=0,TIB_CRIT_BATCH_FACTOR=24 TIB_BATCH_CHAIN=0,TIB_CRIT_BATCH_FACTOR=0 > gpurun_out/r33/ab.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r33/tests.log 2>&1
timeout 400 python bench.py --config batch --no-cpu-baseline --steps 3 > gpurun_out/r33/bench_batch.json 2>&1
