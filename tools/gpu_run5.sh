cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r5
timeout 600 python -m pytest tests/test_configs.py -m gpu -q -p no:cacheprovider -k "device_generator or large or batch_config" > gpurun_out/r5/tests.log 2>&1
timeout 600 python tools/e2e_timing.py large > gpurun_out/r5/timing_large.log 2>&1
timeout 600 python tools/e2e_timing.py batch > gpurun_out/r5/timing_batch.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"rowsum|fill_kernel" -c 4 --csv --log-file gpurun_out/r5/gen.csv python tools/e2e_timing.py large > gpurun_out/r5/ncu_gen.log 2>&1
