cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r36
timeout 300 python tools/e2e_timing.py batch > gpurun_out/r36/batch_e2e.log 2>&1
timeout 400 python bench.py --config batch --no-cpu-baseline --steps 3 > gpurun_out/r36/bench_batch.json 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r36/tests.log 2>&1
