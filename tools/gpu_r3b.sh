cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r3b
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r3b/tests.log 2>&1
for c in batch large kronecker; do
  timeout 900 python tools/ab_env.py $c TIB_UPD_GROUP=1 TIB_UPD_GROUP=2 TIB_UPD_GROUP=3 TIB_UPD_GROUP=4 --rounds 2 > gpurun_out/r3b/ab_$c.log 2>&1
done
