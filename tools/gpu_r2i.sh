cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2i
timeout 1200 python tools/ab_env.py large TIB_C0_PF_P2=0 TIB_C0_PF_P2=1 --rounds 2 > gpurun_out/r2i/ab_large.log 2>&1
timeout 1200 python tools/ab_env.py kronecker TIB_C0_PF_P2=0 TIB_C0_PF_P2=1 > gpurun_out/r2i/ab_kron.log 2>&1
