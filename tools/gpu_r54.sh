cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r54
timeout 900 python -m pytest tests/test_configs.py -m gpu -q -p no:cacheprovider -k kronecker > gpurun_out/r54/tests.log 2>&1
timeout 600 python bench.py --config kronecker --no-cpu-baseline --steps 3 > gpurun_out/r54/bench_kronecker.json 2>&1
