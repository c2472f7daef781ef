cd $GRAFT_REPO_ROOT
O=gpurun_out/r3i
mkdir -p $O
timeout 900 python tools/ab_env.py large TIB_EARLY_TICKET=0 TIB_EARLY_TICKET=1 --rounds 2 > $O/ab_large.log 2>&1
timeout 900 python tools/ab_env.py batch TIB_EARLY_TICKET=0 TIB_EARLY_TICKET=1 --rounds 1 > $O/ab_batch.log 2>&1
timeout 900 python tools/ab_env.py medium TIB_EARLY_TICKET=0 TIB_EARLY_TICKET=1 --rounds 1 > $O/ab_medium.log 2>&1
TIB_EARLY_TICKET=1 timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/tests.log 2>&1
