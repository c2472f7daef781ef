cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/s2j
for cfg in "" "TIB_SOLO_CRIT=1" "TIB_SOLO_CRIT=1 TIB_CRIT_WORKERS_FACTOR=40" "TIB_SOLO_CRIT=1 TIB_CRIT_WORKERS_FACTOR=72" "TIB_CRIT_WORKERS_FACTOR=80"; do
  echo "== $cfg" >> gpurun_out/s2j/runs.log
  env $cfg timeout 300 python tools/prof_run.py large 3 >> gpurun_out/s2j/runs.log 2>&1
done
