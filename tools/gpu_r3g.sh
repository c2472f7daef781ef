cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r3g
timeout 900 python tools/ab_env.py large TIB_CRIT_SPLIT_FACTOR=8 TIB_CRIT_SPLIT_FACTOR=12 TIB_CRIT_SPLIT_FACTOR=16 TIB_CRIT_SPLIT_FACTOR=24 --rounds 1 > gpurun_out/r3g/ab_large_crit.log 2>&1
timeout 900 python tools/ab_env.py medium TIB_CRIT_SPLIT_FACTOR=12 TIB_CRIT_SPLIT_FACTOR=16 TIB_CRIT_SPLIT_FACTOR=24 TIB_CRIT_SPLIT_FACTOR=32 --rounds 1 > gpurun_out/r3g/ab_medium_crit.log 2>&1
timeout 900 python tools/ab_env.py batch TIB_CRIT_BATCH_FACTOR=16 TIB_CRIT_BATCH_FACTOR=24 TIB_CRIT_BATCH_FACTOR=32 TIB_CRIT_BATCH_FACTOR=48 --rounds 1 > gpurun_out/r3g/ab_batch_crit.log 2>&1
timeout 900 python tools/ab_env.py kronecker TIB_CRIT_TPUT_FACTOR=4 TIB_CRIT_TPUT_FACTOR=8 TIB_CRIT_TPUT_FACTOR=12 --rounds 1 > gpurun_out/r3g/ab_kron_crit.log 2>&1
