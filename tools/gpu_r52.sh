cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r52
timeout 1500 python tools/ab_env.py large TIB_SPLIT=1 TIB_DEDICATE_MAX_BATCH=1 TIB_AGENT=0 TIB_POLL_SHIFT=1 --rounds 2 > gpurun_out/r52/ab.log 2>&1
timeout 900 python tools/ab_env.py medium TIB_SPLIT=1 TIB_DEDICATE_MAX_BATCH=1 > gpurun_out/r52/ab_medium.log 2>&1
