cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r61
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r61/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r61/tests.log 2>&1
timeout 600 python bench.py > gpurun_out/r61/bench_large.json 2> gpurun_out/r61/bench_large.err
timeout 600 python bench.py --config medium --no-cpu-baseline > gpurun_out/r61/bench_medium.json 2>&1
