cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2x
timeout 2000 python tools/ab_env.py large TIB_SPLIT=1 TIB_BOUNDARY=0 TIB_DEFER_W=4 TIB_DEFER_W=1 TIB_CRIT_SPLIT_FACTOR=16 TIB_CRIT_SPLIT_FACTOR=32 TIB_FAT_LEAF=1 --rounds 2 > gpurun_out/r2x/ab.log 2>&1
