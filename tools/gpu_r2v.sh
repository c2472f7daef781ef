cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2v
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r2v/tests.log 2>&1
timeout 300 python tools/e2e_timing.py batch > gpurun_out/r2v/batch.log 2>&1
timeout 400 python bench.py --config batch --no-cpu-baseline --steps 3 > gpurun_out/r2v/bench_batch.json 2>&1
