cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2b
timeout 600 python tools/split_probe.py > gpurun_out/r2b/split.log 2>&1
timeout 400 python bench.py --config batch --tile 256 --no-cpu-baseline --steps 3 > gpurun_out/r2b/batch256.json 2>&1
