cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2d
timeout 300 python bench.py --no-cpu-baseline --steps 3 > gpurun_out/r2d/bench_large.json 2>&1
timeout 900 python tools/crit_sweep.py batch 8,24 0,24 8,40 8,56 16,32 0,40 > gpurun_out/r2d/crit_batch.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2d/tests.log 2>&1
