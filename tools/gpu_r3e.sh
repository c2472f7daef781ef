cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r3e
timeout 900 python tools/ab_env.py batch TIB_P2_GROUP=6 TIB_P2_GROUP=8 TIB_P2_GROUP=12 --rounds 1 > gpurun_out/r3e/ab_batch_p2.log 2>&1
timeout 900 python tools/ab_env.py kronecker TIB_P2_GROUP=3 TIB_P2_GROUP=4 --rounds 1 > gpurun_out/r3e/ab_kron_p2.log 2>&1
timeout 900 python tools/ab_env.py large TIB_SPLIT=0 --rounds 1 > gpurun_out/r3e/ab_large_nat.log 2>&1
bash tools/trace_run.sh large > gpurun_out/r3e/trace.log 2>&1
cp gpurun_out/tr/report_large.txt gpurun_out/r3e/ 2>/dev/null
