# task trace of the batch config (64 matrices, one launch per sweep)
mkdir -p gpurun_out/tr /tmp/tibtr
rm -f /tmp/tibtr/*.bin
cat > /tmp/tibtr/runb.py <<'PY'
import sys, os
sys.path.insert(0, ".")
import paper_2504_19171_b200 as tib
ms = [tib.generate(50000, 500, 50, 1.0, seed=1000 + k, tile_size=128, device=0) for k in range(64)]
r = tib.Resident(ms, device=0); r.run(1)
PY
TIB_TRACE=/tmp/tibtr/batch timeout 600 python /tmp/tibtr/runb.py > /dev/null 2>&1
for f in /tmp/tibtr/batch.*.bin; do python tools/trace_report.py $f; done > gpurun_out/tr/report_batch.txt 2>&1
rm -f /tmp/tibtr/*.bin
