# round-2 measurement set (run under gpurun)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2/smi.txt
lscpu > gpurun_out/r2/lscpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2/gpu_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r2/gpu_tests.log
timeout 900 python bench.py --config kronecker --steps 3 --warmup 2 > gpurun_out/r2/bench_kron.json 2> gpurun_out/r2/bench_kron.err
timeout 900 python bench.py --config batch --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/r2/bench_batch.json 2> gpurun_out/r2/bench_batch.err
TIB_BENCH_SAME_DEVICE=1 TIB_BENCH_BACKEND=gloo timeout 900 python bench.py --gpus 2 --config batch --steps 3 --warmup 2 > gpurun_out/r2/bench_batch_2ranks_1gpu.json 2> gpurun_out/r2/bench_batch_2ranks.err
timeout 900 python bench.py --impl reference --config large --ref-full > gpurun_out/r2/ref_large_full.json 2> gpurun_out/r2/ref_large_full.err
timeout 900 python bench.py --impl reference --config batch --ref-throughput > gpurun_out/r2/ref_batch_throughput.json 2> gpurun_out/r2/ref_batch_tp.err
timeout 900 ncu --set full --import-source on --clock-control none -k regex:dataflow -s 1 -c 1 \
  -o gpurun_out/r2/phase2_large python tools/prof_run.py large 1 > gpurun_out/r2/ncu_p2.log 2>&1
ls -la gpurun_out/r2
