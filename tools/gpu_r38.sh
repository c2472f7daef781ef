cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r38
timeout 2000 python tools/ab_env.py large TIB_SPLIT=1 TIB_CRIT_SPLIT_P2=12 TIB_CRIT_SPLIT_P2=40 TIB_CRIT_SPLIT_FACTOR=16 TIB_CRIT_SPLIT_FACTOR=16,TIB_CRIT_SPLIT_P2=40 --rounds 2 > gpurun_out/r38/ab.log 2>&1
