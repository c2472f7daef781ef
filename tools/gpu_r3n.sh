cd $GRAFT_REPO_ROOT
O=gpurun_out/r3n
mkdir -p $O
timeout 1200 python tools/ab_env.py large TIB_SPLIT=0 TIB_SPLIT=0,TIB_CRIT_WORKERS_P2=6 TIB_SPLIT=0,TIB_CRIT_WORKERS_P2=20 TIB_SPLIT=0,TIB_CRIT_WORKERS_P2=32 TIB_SPLIT=0,TIB_UPD_GROUP=2 --rounds 1 > $O/ab_large_nat.log 2>&1
