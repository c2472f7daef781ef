cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/final2
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > gpurun_out/final2/smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final2/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/final2/tests.log 2>&1
timeout 600 python bench.py > gpurun_out/final2/bench_large.json 2> gpurun_out/final2/bench_large.err
for c in medium batch kronecker; do
  timeout 600 python bench.py --config $c > gpurun_out/final2/bench_$c.json 2> gpurun_out/final2/bench_$c.err
done
timeout 900 python bench.py --impl reference > gpurun_out/final2/ref_large.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final2/launches_smoke.csv python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final2/smoke_ncu.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final2/launches_bench.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/final2/bench_ncu.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:dataflow_kernel --launch-skip 1 -c 1 -o gpurun_out/final2/phase2_large python tools/prof_run.py large 1 > gpurun_out/final2/ncu_p2.log 2>&1
