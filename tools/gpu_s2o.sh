cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/s2o
timeout 300 python tools/e2e_timing.py kronecker > gpurun_out/s2o/kron.log 2>&1
timeout 300 python tools/e2e_probe.py large > gpurun_out/s2o/large.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/s2o/tests.log 2>&1
