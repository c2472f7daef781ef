# round-2 final measurements (session 4, after the chunk-count hint and batch early tickets): bench lines, reference arm, launch lists, ncu of both sweeps
cd $GRAFT_REPO_ROOT
O=gpurun_out/final4
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > $O/smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/tests.log 2>&1
timeout 600 python bench.py > $O/bench_large.json 2> $O/bench_large.err
for c in medium batch kronecker; do
  timeout 600 python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 900 python bench.py --impl reference > $O/ref_large.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_smoke.csv python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_ncu.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_bench.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $O/bench_ncu.log 2>&1
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:dataflow_kernel -c 1 -o $O/factor_large python tools/prof_run.py large 1 > $O/ncu_factor.log 2>&1
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:dataflow_kernel --launch-skip 1 -c 1 -o $O/phase2_large python tools/prof_run.py large 1 > $O/ncu_p2.log 2>&1
