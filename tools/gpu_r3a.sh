cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r3a
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > gpurun_out/r3a/smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3a/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r3a/tests.log 2>&1
timeout 600 python bench.py > gpurun_out/r3a/bench_large.json 2> gpurun_out/r3a/bench_large.err
