cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2k
for st in 8 4 2 0 8 4 2 0; do
  TIB_DIAG_STRIPS=$st timeout 300 python bench.py --no-cpu-baseline --steps 3 > gpurun_out/r2k/bench_s$st.json 2>&1
  echo "strips $st $(python tools/bsum.py gpurun_out/r2k/bench_s$st.json)" >> gpurun_out/r2k/strips.log
done
