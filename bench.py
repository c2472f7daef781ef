#!/usr/bin/env python
"""Benchmark of the B200 tile Cholesky + selected inversion (arXiv 2504.19171 hot path).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config large]

One step = one fused factorize + selected inversion ("pattern": every tile of
L's pattern, marginal variances and logdet included) of one synthetic
arrowhead matrix of the BASELINE configuration, generated bit-exactly like
the reference generator (density 1, seed 42 + rank).  Multi-GPU (torchrun,
one process per GPU): independent matrices per rank (an INLA-style batch
sharded over GPUs) -- weak scaling, no data-path collective; the barrier and
the MAX-over-ranks time reduction use torch.distributed (NCCL).

metric: FP64 TFLOP/s under the reference's task model,
whole job.  `value` is device time (CUDA events on the library stream) with
the matrix resident in HBM; `e2e` goes through the public API
(paper_2504_19171_b200.selected_inverse + .diagonal() + .logdet()) from the
pinned host matrix, host->device copy and the marginal-variance read-back
inside the timed region.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (n, bandwidth, thickness, tile)   -- BASELINE.json configs
    "small": (10000, 200, 50, 128),
    "medium": (100000, 1000, 100, 256),
    "large": (200000, 2000, 200, 512),
    "batch": (50000, 500, 50, 128),  # BASELINE config 5: 64 such matrices, split over the GPUs
}
BATCH_TOTAL = {"batch": 64}  # matrices per step over all GPUs (config 5, seeds 1000..1063)
METRIC = "factorize+selinv FP64 TFLOP/s (reference task model), whole job"
PEAK_FILE = os.path.join(ROOT, "profiles", "r01_fp64_peak.jsonl")
TRAFFIC_FILE = os.path.join(ROOT, "profiles", "dataflow_traffic.json")
REF_DRIVER = os.path.join(ROOT, "oracle", "_ref", "ref_driver")
REF_SAMPLE_N = {"small": 10000, "medium": 12000, "large": 12000, "batch": 50000}  # bounded CPU sample (same w, t, b)


def fp64_peak():
    """Measured FP64 DMMA peak on this pool's B200 (tools/fp64_peak.cu ->
    profiles/r01_fp64_peak.jsonl); MEASURED_PEAKS.json carries no FP64 entry."""
    try:
        rows = [json.loads(line) for line in open(PEAK_FILE) if line.strip().startswith("{")]
        sus = [r["tflops"] for r in rows if r.get("kind") == "dmma_sustained_4s"]
        return sus[0], "measured in-repo: DMMA m8n8k4 sustained 4 s (profiles/r01_fp64_peak.jsonl)"
    except (OSError, ValueError, IndexError, KeyError):
        return 37.0, "fallback: nominal HGX B200 FP64 tensor 37 TFLOP/s"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.rows = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                if out.returncode == 0 and out.stdout.strip():
                    self.rows.append([x.strip() for x in out.stdout.strip().split(",")])
            except (OSError, subprocess.SubprocessError):
                return
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 4 + i and r[4 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows),
                "power_w_max": max((float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()), default=None)}


def ref_bench(n, w, t, b, seed, workers):
    out = subprocess.run([REF_DRIVER, "bench", str(n), str(w), str(t), str(b), str(seed), str(workers)],
                         check=True, capture_output=True, text=True).stdout
    return json.loads(out)


def cpu_baseline(cfg_name, w, t, b):
    """The reference CPU path (oracle/_ref, built from /root/reference/proj by
    oracle/Makefile) on the box's host cores, on a bounded sample of the same
    workload: same bandwidth, arrow and tile size, fewer tile columns."""
    cores = os.cpu_count() or 1
    n = REF_SAMPLE_N[cfg_name]
    if os.path.exists(REF_DRIVER):
        r = ref_bench(n, w, t, b, 42, cores)
        return {"value": r["gflop"] / r["total_s"] / 1e3, "unit": "TFLOP/s", "cores": cores, "kind": "reference",
                "sample": f"n={n} w={w} t={t} b={b} seed 42 ({r['N']} tile columns), factorize+phase1+phase2, "
                          f"workers={cores}, {r['total_s']:.2f} s"}
    from oracle import oracle as orc  # CPU port (single thread) when the reference build is absent

    t0 = time.perf_counter()
    orc.selected_inverse_generated(n, w, t, 1.0, 42, b, "pattern")
    dt = time.perf_counter() - t0
    import paper_2504_19171_b200 as tib

    fl = sum(tib.task_flops(tib.generate(n, w, t, 1.0, seed=42, tile_size=b)))
    return {"value": fl / dt / 1e12, "unit": "TFLOP/s", "cores": 1, "kind": "port",
            "sample": f"n={n} w={w} t={t} b={b} seed 42, oracle/tileinv_oracle.c single thread"}


def run_reference(args, rank, world):
    """--impl reference: the reference's own CPU implementation of the path
    (oracle/_ref/ref_driver over libtileinv_core), all host threads, one
    bounded sample of the workload per step; rank 0 only."""
    if rank != 0:
        return
    n, w, t, b = CONFIGS[args.config]
    cores = os.cpu_count() or 1
    ns = REF_SAMPLE_N[args.config]
    if not os.path.exists(REF_DRIVER):
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built (needs /root/reference at build)"}))
        return
    for _ in range(args.warmup):
        ref_bench(ns, w, t, b, 42, cores)
    rates, secs = [], []
    for _ in range(args.steps):
        r = ref_bench(ns, w, t, b, 42, cores)
        rates.append(r["gflop"] / r["total_s"] / 1e3)
        secs.append(r["total_s"])
    value = statistics.median(rates)
    sample = f"n={ns} w={w} t={t} b={b} seed 42 per step (same band/arrow/tile as the workload), workers={cores}"
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * statistics.median(secs),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference generator, density 1, seed 42)",
        "config": {"workload": f"{args.config} arrowhead n={n} w={w} t={t} b={b}: factorize + selected inversion "
                               f"(pattern), reference CPU path on a bounded sample", "sample_n": ns, "n": n,
                   "bandwidth": w, "thickness": t, "tile": b},
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": cores, "kind": "reference", "sample": sample},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="large", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        if dist:
            dist.barrier()

    def max_over_ranks(x):
        if not dist:
            return x
        tt = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        return float(tt.item())

    import paper_2504_19171_b200 as tib

    n, w, t, b = CONFIGS[args.config]
    per = max(1, BATCH_TOTAL.get(args.config, world) // world)  # matrices per GPU per step
    if args.config in BATCH_TOTAL:
        ms = [tib.generate(n, w, t, 1.0, seed=1000 + rank * per + k, tile_size=b) for k in range(per)]
    else:
        ms = [tib.generate(n, w, t, 1.0, seed=42 + rank, tile_size=b)]
    m = ms[0]
    f_fact, f_p1, f_p2 = tib.task_flops(m)
    flops = (f_fact + f_p1 + f_p2) * per  # per GPU per step
    _, _, stored_tiles = m.n, m.tile_size, m.stored_tiles
    h2d = stored_tiles * b * b * 8 * per
    d2h = n * 8 * per

    # ---- device-resident timing: K fused sweeps, CUDA events on the library stream
    res = tib.Resident(m if per == 1 else ms, device=local)
    res.run(args.warmup)
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        tot_ms, ms_fact, ms_p2 = res.run(args.steps)
        torch.cuda.synchronize()
    barrier()
    info = res.info()
    del res
    ms_step = max_over_ranks(tot_ms / args.steps)
    value = world * flops / (ms_step / 1e3) / 1e12

    # ---- end to end through the public API, host buffers, H2D + D2H inside
    def public_call():
        if per == 1:
            r = tib.selected_inverse(m, "pattern", device=local)
            _ = r.diagonal(), r.logdet()
            del r
        else:  # marginal variances + logdet of every matrix of the batch, one batched call
            _ = tib.selected_inverse_batch(ms, device=local)

    public_call()
    torch.cuda.synchronize()
    barrier()
    t0 = time.perf_counter()
    e2e_steps = max(1, min(args.steps, 3))
    for _ in range(e2e_steps):
        public_call()
    torch.cuda.synchronize()
    e2e_s = max_over_ranks((time.perf_counter() - t0) / e2e_steps)
    barrier()
    e2e = world * flops / e2e_s / 1e12

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return
    peak, peak_src = fp64_peak()
    per_gpu = flops / (ms_step / 1e3) / 1e12
    traffic = None
    try:
        traffic = json.load(open(TRAFFIC_FILE)).get(args.config)
    except (OSError, ValueError):
        pass
    line = {
        "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong" if args.config in BATCH_TOTAL else "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (bit-exact reference generator, density 1, " +
                ("seeds 1000..1063 over the GPUs)" if args.config in BATCH_TOTAL else "seed 42+rank)"),
        "config": {"workload": f"{args.config} arrowhead n={n} w={w} t={t} b={b}"
                               + (f" x{per} matrices per GPU (one batched launch per sweep)" if per > 1 else "")
                               + ": fused factorize + selected inversion (pattern) + marginal variances + logdet "
                                 "per matrix",
                   "n": n, "bandwidth": w, "thickness": t, "tile": b, "matrices_per_gpu_per_step": per,
                   "parallelism": f"independent matrices per GPU (x{world})",
                   "l2": "inputs larger than L2 (tile store %.1f GB per copy)" % (h2d / 1e9),
                   "task_model_gflop": flops / 1e9, "executed_gflop": info["executed_flops"] / 1e9},
        "seconds_per_matrix": ms_step / 1e3 / per,
        "ms_factorize_sweep": ms_fact, "ms_phase2_sweep": ms_p2,
        "logdet": info["logdet"],
        "e2e": {"value": e2e, "unit": "TFLOP/s", "h2d_bytes_per_step": h2d * world, "d2h_bytes_per_step": d2h * world,
                "seconds_per_matrix": e2e_s / per},
        "gpu_launches": int(info["kernel_launches_per_rep"]) * args.steps,
        "roofline": {"bound": "tensor", "achieved": per_gpu, "peak": peak, "unit": "TFLOP/s",
                     "frac": per_gpu / peak, "traffic": traffic, "peak_source": peak_src,
                     "kernel": "dataflow_kernel (both sweeps; task-model FLOPs / event time)"},
        "clocks": clk.summary(),
    }
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args.config, w, t, b)
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
