cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2f
for c in 56 24 8; do
  for k in 2 4; do
    TIB_CRIT_WORKERS_FACTOR=$c timeout 300 python tools/split_probe.py $k > gpurun_out/r2f/split_${k}_$c.log 2>&1
  done
done
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -k "generator or batch" > gpurun_out/r2f/tests.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2f/gen_launches.csv python tools/gen_probe.py 1 > gpurun_out/r2f/gen.log 2>&1
timeout 300 python bench.py --no-cpu-baseline --steps 3 > gpurun_out/r2f/bench_large.json 2>&1
