cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r3
timeout 600 python tools/e2e_timing.py batch > gpurun_out/r3/timing_batch.log 2>&1
timeout 600 python tools/e2e_timing.py kronecker > gpurun_out/r3/timing_kron.log 2>&1
timeout 600 python tools/e2e_timing.py large > gpurun_out/r3/timing_large.log 2>&1
TIB_STREAM_UPLOAD=0 timeout 600 python tools/e2e_timing.py batch > gpurun_out/r3/timing_batch_nostream.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_configs.py -m gpu -q -p no:cacheprovider -k "kron or batch or stream" > gpurun_out/r3/tests.log 2>&1
