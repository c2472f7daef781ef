cd $GRAFT_REPO_ROOT
O=gpurun_out/r3j
mkdir -p $O
TIB_PREFETCH=1 TIB_WATCHDOG_S=20 timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 900 python tools/ab_env.py large TIB_PREFETCH=0 TIB_PREFETCH=1 --rounds 2 > $O/ab_large.log 2>&1
timeout 900 python tools/ab_env.py batch TIB_PREFETCH=0 TIB_PREFETCH=1 --rounds 1 > $O/ab_batch.log 2>&1
timeout 900 python tools/ab_env.py medium TIB_PREFETCH=0 TIB_PREFETCH=1 --rounds 1 > $O/ab_medium.log 2>&1
timeout 900 python tools/ab_env.py kronecker TIB_PREFETCH=0 TIB_PREFETCH=1 --rounds 1 > $O/ab_kron.log 2>&1
TIB_PREFETCH=1 TIB_WATCHDOG_S=20 timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/tests.log 2>&1
