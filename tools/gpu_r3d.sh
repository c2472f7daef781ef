cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r3d
timeout 900 python tools/ab_env.py large TIB_SPLIT=0,TIB_UPD_GROUP=1 TIB_SPLIT=0,TIB_UPD_GROUP=4 --rounds 1 > gpurun_out/r3d/ab_large_nat.log 2>&1
timeout 900 python tools/ab_env.py batch TIB_P2_GROUP=3 TIB_P2_GROUP=4 TIB_P2_GROUP=6 --rounds 1 > gpurun_out/r3d/ab_batch_p2.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r3d/tests.log 2>&1
timeout 600 python bench.py > gpurun_out/r3d/bench_large.json 2> gpurun_out/r3d/bench_large.err
for c in medium batch kronecker; do
  timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/r3d/bench_$c.json 2> gpurun_out/r3d/bench_$c.err
done
