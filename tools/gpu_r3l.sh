cd $GRAFT_REPO_ROOT
O=gpurun_out/r3l
mkdir -p $O
timeout 1200 python tools/ab_env.py large TIB_POLL_SHIFT=0 TIB_POLL_SHIFT=1 TIB_COARSE_SECOND=0 TIB_P2_GROUP=2 TIB_CRIT_SPLIT_P2=16 TIB_CRIT_SPLIT_P2=8 --rounds 1 > $O/ab_large.log 2>&1
timeout 900 python tools/ab_env.py medium TIB_POLL_SHIFT=0 TIB_POLL_SHIFT=1 TIB_CRIT_SPLIT_P2=32 --rounds 1 > $O/ab_medium.log 2>&1
