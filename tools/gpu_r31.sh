cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r31
for i in 1 2; do
timeout 300 python bench.py --no-cpu-baseline --steps 3 > gpurun_out/r31/bench_def$i.json 2>&1
TIB_P2_GROUP=1 timeout 300 python bench.py --no-cpu-baseline --steps 3 > gpurun_out/r31/bench_g1_$i.json 2>&1
done
timeout 900 python tools/ab_env.py large TIB_SPLIT=0,TIB_P2_GROUP=1 TIB_SPLIT=0,TIB_P2_GROUP=3 TIB_SPLIT=0,TIB_P2_GROUP=2 > gpurun_out/r31/ab.log 2>&1
