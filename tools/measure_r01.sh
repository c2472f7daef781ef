# Round-1 measurement set (run under gpurun): bench line, ncu launch list of the
# bench command, one ncu --set full capture of the factor sweep (large).
set -x
mkdir -p gpurun_out/m
timeout 500 python bench.py > gpurun_out/m/bench.json 2> gpurun_out/m/bench.err
timeout 600 python bench.py --config batch > gpurun_out/m/bench_batch.json 2> gpurun_out/m/bench_batch.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv \
  --log-file gpurun_out/m/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/m/ncu_bench.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:dataflow -c 1 \
  -o gpurun_out/m/dataflow_large python tools/prof_run.py large 1 > gpurun_out/m/ncu_full.log 2>&1
ls -la gpurun_out/m
