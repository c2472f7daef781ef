# traces of the public call's factor sweep (streamed upload): natural and two-chain order
mkdir -p gpurun_out/tr /tmp/tibtr
rm -f /tmp/tibtr/*.bin
cat > /tmp/tibtr/run.py <<'PY'
import sys, os
sys.path.insert(0, ".")
import paper_2504_19171_b200 as tib
m = tib.generate(200000, 2000, 200, 1.0, seed=42, tile_size=512)
r = tib.selected_inverse(m, "pattern"); del r
os.environ["TIB_TRACE"] = sys.argv[1]
r = tib.selected_inverse(m, "pattern"); del r
PY
timeout 300 python /tmp/tibtr/run.py /tmp/tibtr/nat > /dev/null 2>&1
TIB_SPLIT_STREAMED=1 timeout 300 python /tmp/tibtr/run.py /tmp/tibtr/ss > /dev/null 2>&1
ls /tmp/tibtr > gpurun_out/tr/e2e_files.txt
for f in /tmp/tibtr/nat.0.bin /tmp/tibtr/ss.0.bin; do python tools/trace_report.py $f; done > gpurun_out/tr/report_e2e.txt 2>&1
rm -f /tmp/tibtr/*.bin
