cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r3f
timeout 900 python tools/ab_env.py large TIB_UPD_GROUP=4 TIB_UPD_GROUP=8 --rounds 1 > gpurun_out/r3f/ab_large.log 2>&1
timeout 900 python tools/ab_env.py medium TIB_UPD_GROUP=4 --rounds 1 > gpurun_out/r3f/ab_medium.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r3f/tests.log 2>&1
bash tools/trace_run.sh large > gpurun_out/r3f/trace.log 2>&1
cp gpurun_out/tr/report_large.txt gpurun_out/r3f/ 2>/dev/null
