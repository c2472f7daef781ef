# round-2 session-2 validation of HEAD: full GPU suite, smoke, bench (large, default), launch list
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/s2a
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/s2a/smi.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/s2a/gpu_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/s2a/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s2a/smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/s2a/smoke.log
timeout 900 python bench.py > gpurun_out/s2a/bench.json 2> gpurun_out/s2a/bench.err
timeout 600 python bench.py --config batch --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/s2a/bench_batch.json 2> gpurun_out/s2a/bench_batch.err
