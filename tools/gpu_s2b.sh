# chain diagnostics: phase profile (prof build), task trace report, leaf / latency microbenchmarks
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/s2b
TIB_LIB_VARIANT=prof TIB_CHAIN_PROF=1 timeout 300 python tools/prof_run.py large 1 > gpurun_out/s2b/chainprof_large.log 2>&1
TIB_LIB_VARIANT=prof TIB_CHAIN_PROF=1 timeout 300 python tools/prof_run.py mini 1 > gpurun_out/s2b/chainprof_mini.log 2>&1
bash tools/trace_run.sh large > gpurun_out/s2b/trace_run.log 2>&1
cp gpurun_out/tr/report_large.txt gpurun_out/s2b/ 2>/dev/null
cd tools
for b in leaf_bench lat_bench; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2504_19171_b200/csrc $b.cu -o /tmp/$b > ../gpurun_out/s2b/$b.build 2>&1 && timeout 60 /tmp/$b > ../gpurun_out/s2b/$b.log 2>&1
done
