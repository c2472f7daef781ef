"""Summarise an ncu --set full report (first kernel) into a small JSON for profiles/.

    python tools/ncu_summary.py gpurun_out/x.ncu-rep profiles/r02_x.json [label]
"""
import csv
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "lts__t_sector_hit_rate.pct",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
]


def main():
    rep, out = sys.argv[1], sys.argv[2]
    label = sys.argv[3] if len(sys.argv) > 3 else rep
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2]
    res = {"report": rep, "label": label, "kernel": vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else None}
    for k in KEYS:
        if k in hdr:
            i = hdr.index(k)
            res[k] = {"value": vals[i], "unit": units[i]}
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
