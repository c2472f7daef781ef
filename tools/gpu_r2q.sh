cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2q
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2q/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2q/tests.log 2>&1
timeout 300 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/r2q/bench_large.json 2>&1
timeout 300 python bench.py --config medium --no-cpu-baseline --steps 5 > gpurun_out/r2q/bench_medium.json 2>&1
timeout 400 python bench.py --config kronecker --no-cpu-baseline --steps 3 > gpurun_out/r2q/bench_kron.json 2>&1
