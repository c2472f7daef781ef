cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r55
timeout 1500 python tools/ab_env.py medium TIB_SPLIT=1 TIB_CRIT_SPLIT_FACTOR=32 TIB_CRIT_SPLIT_FACTOR=48 TIB_CRIT_SPLIT_P2=24 TIB_CRIT_SPLIT_P2=4 --rounds 2 > gpurun_out/r55/ab.log 2>&1
timeout 1200 python tools/ab_env.py batch TIB_SPLIT=1 TIB_CRIT_BATCH_P2=24 TIB_CRIT_BATCH_P2=64 > gpurun_out/r55/ab_batch.log 2>&1
