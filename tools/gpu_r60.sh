cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r60
timeout 2400 python tools/ab_env.py large TIB_COARSE_SECOND=0 TIB_COARSE_SECOND=1 --rounds 2 > gpurun_out/r60/ab.log 2>&1
timeout 900 python tools/ab_env.py medium TIB_COARSE_SECOND=0 TIB_COARSE_SECOND=1 > gpurun_out/r60/ab_medium.log 2>&1
