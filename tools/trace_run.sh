# usage: bash tools/trace_run.sh <config> [tag]; env vars pass through (e.g. TIB_FAT_LEAF=1)
# traces go to /tmp on the box; the report to gpurun_out/tr/report_<config><tag>.txt
cfg=${1:-large}
tag=${2:-}
mkdir -p gpurun_out/tr /tmp/tibtr
rm -f /tmp/tibtr/*.bin
TIB_TRACE=/tmp/tibtr/$cfg$tag timeout 300 python tools/prof_run.py $cfg 1 > /dev/null
timeout 300 python tools/prof_run.py $cfg 3
for f in /tmp/tibtr/$cfg$tag.*.bin; do python tools/trace_report.py $f; done > gpurun_out/tr/report_$cfg$tag.txt 2>&1
rm -f /tmp/tibtr/*.bin
