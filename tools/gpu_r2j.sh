cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2j
timeout 1500 python tools/ab_env.py large TIB_C0_PF_FACTOR=0 TIB_C0_PF_FACTOR=1 TIB_LIB_VARIANT=old --rounds 2 > gpurun_out/r2j/ab_large3.log 2>&1
