cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2z
timeout 1500 python tools/ab_env.py large TIB_P2_GROUP=1 TIB_P2_GROUP=2 TIB_P2_GROUP=3 TIB_P2_GROUP=5 --rounds 2 > gpurun_out/r2z/ab_large.log 2>&1
timeout 900 python tools/ab_env.py kronecker TIB_P2_GROUP=1 TIB_P2_GROUP=2 TIB_P2_GROUP=3 > gpurun_out/r2z/ab_kron.log 2>&1
timeout 900 python tools/ab_env.py batch TIB_P2_GROUP=1 TIB_P2_GROUP=2 TIB_P2_GROUP=3 > gpurun_out/r2z/ab_batch.log 2>&1
timeout 900 python tools/ab_env.py medium TIB_P2_GROUP=1 TIB_P2_GROUP=2 TIB_P2_GROUP=3 > gpurun_out/r2z/ab_medium.log 2>&1
