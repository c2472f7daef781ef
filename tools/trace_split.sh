# trace of the two-chain probe (2 x n=100200, one launch)
mkdir -p gpurun_out/tr /tmp/tibtr
rm -f /tmp/tibtr/*.bin
TIB_CRIT_WORKERS_FACTOR=24 TIB_TRACE=/tmp/tibtr/split2 timeout 300 python tools/split_probe.py 2 > /dev/null
for f in /tmp/tibtr/split2.*.bin; do python tools/trace_report.py $f; done > gpurun_out/tr/report_split2.txt 2>&1
rm -f /tmp/tibtr/*.bin
