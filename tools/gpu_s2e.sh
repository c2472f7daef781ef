cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/s2e
for b in sweep_bench chain_bench leaf_bench; do timeout 60 tools/bin/$b > gpurun_out/s2e/$b.log 2>&1; done
