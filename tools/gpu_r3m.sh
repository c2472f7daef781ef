cd $GRAFT_REPO_ROOT
O=gpurun_out/r3m
mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/tests.log 2>&1
timeout 600 python bench.py > $O/bench_large.json 2> $O/bench_large.err
timeout 600 python bench.py --config medium > $O/bench_medium.json 2> $O/bench_medium.err
