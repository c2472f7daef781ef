# usage: bash tools/trace_run.sh <config> [tag]; env vars pass through (e.g. TIB_FAT_LEAF=1)
# writes gpurun_out/tr/report_<config><tag>.txt
set -e
cfg=${1:-large}
tag=${2:-}
mkdir -p gpurun_out/tr
TIB_TRACE=gpurun_out/tr/$cfg$tag timeout 300 python tools/prof_run.py $cfg 1 > /dev/null
timeout 300 python tools/prof_run.py $cfg 3
for f in gpurun_out/tr/$cfg$tag.*.bin; do python tools/trace_report.py $f; done > gpurun_out/tr/report_$cfg$tag.txt 2>&1
rm -f gpurun_out/tr/*.bin
