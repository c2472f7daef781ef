# usage: bash tools/trace_run.sh <config> [env...]; writes gpurun_out/tr/report_<config>.txt
set -e
cfg=${1:-large}
mkdir -p gpurun_out/tr
TIB_TRACE=gpurun_out/tr/$cfg timeout 300 python tools/prof_run.py $cfg 1 > /dev/null
timeout 300 python tools/prof_run.py $cfg 3
for f in gpurun_out/tr/$cfg.*.bin; do python tools/trace_report.py $f; done > gpurun_out/tr/report_$cfg.txt 2>&1
rm -f gpurun_out/tr/*.bin
