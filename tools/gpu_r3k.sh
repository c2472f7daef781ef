cd $GRAFT_REPO_ROOT
O=gpurun_out/r3k
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k grouped -p no:cacheprovider > $O/tests.log 2>&1
