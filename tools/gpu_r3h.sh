cd $GRAFT_REPO_ROOT
O=gpurun_out/r3h
mkdir -p $O
timeout 900 python tools/ab_env.py kronecker TIB_CRIT_TPUT_FACTOR=4 TIB_CRIT_TPUT_FACTOR=8 TIB_CRIT_TPUT_FACTOR=16 --rounds 1 > $O/ab_kron_crit.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/tests.log 2>&1
timeout 600 python bench.py > $O/bench_large.json 2> $O/bench_large.err
for c in medium kronecker; do
  timeout 600 python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err
done
