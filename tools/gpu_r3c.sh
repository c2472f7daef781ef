cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r3c
for c in batch large kronecker; do
  timeout 900 python tools/ab_env.py $c TIB_UPD_GROUP=4 TIB_UPD_GROUP=6 TIB_UPD_GROUP=8 TIB_UPD_GROUP=16 --rounds 1 > gpurun_out/r3c/ab_$c.log 2>&1
done
timeout 900 python tools/ab_env.py medium TIB_UPD_GROUP=1 TIB_UPD_GROUP=2 TIB_UPD_GROUP=4 --rounds 1 > gpurun_out/r3c/ab_medium.log 2>&1
