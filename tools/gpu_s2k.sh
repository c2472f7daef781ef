cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/s2k
timeout 600 python bench.py --config batch --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/s2k/batch128.json 2> gpurun_out/s2k/batch128.err
timeout 600 python bench.py --config batch --tile 256 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/s2k/batch256.json 2> gpurun_out/s2k/batch256.err
timeout 600 python tools/e2e_timing.py batch > gpurun_out/s2k/timing_batch.log 2>&1
timeout 600 python tools/e2e_timing.py kronecker > gpurun_out/s2k/timing_kron.log 2>&1
