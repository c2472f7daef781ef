cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2a
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2a/smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2a/smoke.log 2>&1
timeout 300 python bench.py > gpurun_out/r2a/bench_large.json 2> gpurun_out/r2a/bench_large.err
timeout 400 python bench.py --config kronecker --no-cpu-baseline > gpurun_out/r2a/bench_kron.json 2> gpurun_out/r2a/bench_kron.err
timeout 400 python bench.py --config batch --no-cpu-baseline > gpurun_out/r2a/bench_batch.json 2> gpurun_out/r2a/bench_batch.err
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2a/tests.log 2>&1
