#!/usr/bin/env python
"""Benchmark of the B200 tile Cholesky + selected inversion (arXiv 2504.19171 hot path).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config large|medium|small|batch|kronecker]

One step = one fused factorize + selected inversion ("pattern": every tile of
L's pattern, marginal variances and logdet included) of the BASELINE
workload: one synthetic arrowhead matrix generated bit-exactly like the
reference generator (density 1, seed 42 + rank), the Kronecker AR1 x SPDE
INLA precision of config 4, or -- `--config batch`, BASELINE config 5 -- the
64-matrix INLA sweep (seeds 1000..1063) sharded over the GPUs.

Multi-GPU: one process per GPU (torchrun; `--gpus N` without a torchrun
environment re-launches itself under torch.distributed.run).  Independent
matrices per rank -- weak scaling for the single-matrix configs, strong
scaling over the 64 matrices of the batch config (shard.batch_seeds) -- and no
data-path collective: the barrier and the MAX-over-ranks time reduction use
torch.distributed (NCCL; TIB_BENCH_BACKEND=gloo for host-side plumbing only).

metric: FP64 TFLOP/s under the reference's task model,
whole job.  `value` is device time (CUDA events on the library stream) with
the matrices resident in HBM; `e2e` goes through the public API
(paper_2504_19171_b200.selected_inverse / selected_inverse_batch +
marginal variances + logdet) from pinned host matrices, host->device copies
and the marginal-variance read-back inside the timed region;
`e2e_device_generated` is the same call on a device-generated matrix
(generate(..., device=k): no host payload, no H2D).
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (n, bandwidth, thickness, tile)   -- BASELINE.json configs (kronecker: n only)
    "small": (10000, 200, 50, 128),
    "medium": (100000, 1000, 100, 256),
    "large": (200000, 2000, 200, 512),
    "batch": (50000, 500, 50, 128),  # BASELINE config 5: 64 such matrices, split over the GPUs
    "kronecker": (200020, None, 20, 512),  # config 4: AR1(50) x SPDE(80 x 50) + 20 fixed effects
}
BATCH_TOTAL = {"batch": 64}  # matrices per step over all GPUs (config 5, seeds 1000..1063)
METRIC = "factorize+selinv FP64 TFLOP/s (reference task model), whole job"
PEAK_FILE = os.path.join(ROOT, "profiles", "r01_fp64_peak.jsonl")
TRAFFIC_FILE = os.path.join(ROOT, "profiles", "dataflow_traffic.json")
REF_DRIVER = os.path.join(ROOT, "oracle", "_ref", "ref_driver")
# bounded CPU sample of each workload for the reference arm: same band, arrow and tile size, fewer tile columns
REF_SAMPLE_N = {"small": 10000, "medium": 12000, "large": 12000, "batch": 50000}
KRON_SAMPLE_NT = 3  # kronecker: 3 of the 50 time steps (n = 12,020), same lattice / fixed effects / tile


def fp64_peak():
    """Measured FP64 DMMA peak on this pool's B200 (tools/fp64_peak.cu ->
    profiles/r01_fp64_peak.jsonl); MEASURED_PEAKS.json carries no FP64 entry."""
    try:
        rows = [json.loads(line) for line in open(PEAK_FILE) if line.strip().startswith("{")]
        sus = [r["tflops"] for r in rows if r.get("kind") == "dmma_sustained_4s"]
        return sus[0], "measured in-repo: DMMA m8n8k4 sustained 4 s (profiles/r01_fp64_peak.jsonl)"
    except (OSError, ValueError, IndexError, KeyError):
        return 37.0, "fallback: nominal HGX B200 FP64 tensor 37 TFLOP/s"


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


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


# ---------------------------------------------------------------------------
# the reference's CPU path (oracle/_ref: the unmodified reference built from
# /root/reference/proj by oracle/Makefile, driven by oracle/ref_driver.cpp)

def ref_bench(n, w, t, b, seed, workers):
    out = subprocess.run([REF_DRIVER, "bench", str(n), str(w), str(t), str(b), str(seed), str(workers)],
                         check=True, capture_output=True, text=True).stdout
    return json.loads(out)


def ref_bench_mm(path, b, workers):
    out = subprocess.run([REF_DRIVER, "bench_mm", path, str(b), str(workers)], check=True, capture_output=True,
                         text=True).stdout
    return json.loads(out)


class RefSample:
    """One bounded sample of a workload for the reference CPU path."""

    def __init__(self, cfg, full=False):
        self.cfg = cfg
        n, w, t, b = CONFIGS[cfg]
        self.b = b
        self.mm = None
        if cfg == "kronecker":
            import paper_2504_19171_b200 as tib

            kc = dict(tib.KRONECKER_CONFIG)
            if not full:
                kc["nt"] = KRON_SAMPLE_NT
            self._tmp = tempfile.TemporaryDirectory()
            self.mm = os.path.join(self._tmp.name, "kron.mtx")
            m = tib.generate_kronecker(tile_size=b, **kc)
            tib.write_matrix_market(m, self.mm)
            self.n = m.n
            self.desc = (f"Kronecker AR1 x SPDE nt={kc['nt']} x {kc['nx']}x{kc['ny']} sites + {kc['p']} fixed "
                         f"effects (n={self.n}) b={b}, read as Matrix Market")
        else:
            self.n = n if full else REF_SAMPLE_N[cfg]
            self.w, self.t = w, t
            self.desc = f"n={self.n} w={w} t={t} b={b} seed 42"

    def run(self, workers):
        if self.mm:
            return ref_bench_mm(self.mm, self.b, workers)
        return ref_bench(self.n, self.w, self.t, self.b, 42, workers)


def cpu_baseline(cfg_name):
    """The reference CPU path on the box's host cores, on a bounded sample of
    the same workload: same bandwidth, arrow and tile size, fewer tile columns."""
    cores = os.cpu_count() or 1
    if os.path.exists(REF_DRIVER):
        s = RefSample(cfg_name)
        r = s.run(cores)
        return {"value": r["gflop"] / r["total_s"] / 1e3, "unit": "TFLOP/s", "cores": cores, "kind": "reference",
                "cpu_model": cpu_model(),
                "sample": f"{s.desc} ({r['N']} tile columns), factorize+phase1+phase2, workers={cores}, "
                          f"{r['total_s']:.2f} s"}
    from oracle import oracle as orc  # CPU port (single thread) when the reference build is absent

    n, w, t, b = CONFIGS[cfg_name]
    n = REF_SAMPLE_N.get(cfg_name, 12000)
    w = w if w is not None else 2000
    t0 = time.perf_counter()
    orc.selected_inverse_generated(n, w, t, 1.0, 42, b, "pattern")
    dt = time.perf_counter() - t0
    import paper_2504_19171_b200 as tib

    fl = sum(tib.task_flops(tib.generate(n, w, t, 1.0, seed=42, tile_size=b)))
    return {"value": fl / dt / 1e12, "unit": "TFLOP/s", "cores": 1, "kind": "port", "cpu_model": cpu_model(),
            "sample": f"n={n} w={w} t={t} b={b} seed 42, oracle/tileinv_oracle.c single thread"}


def run_reference(args, rank, world):
    """--impl reference: the reference's own CPU implementation of the path
    (oracle/_ref/ref_driver over libtileinv_core), all host threads, one
    bounded sample of the workload per step (--ref-full: the whole workload,
    once); rank 0 only.  --ref-throughput (batch): nproc concurrent
    single-thread reference processes, one batch member each."""
    if rank != 0:
        return
    cores = os.cpu_count() or 1
    if not os.path.exists(REF_DRIVER):
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built (needs /root/reference at build)"}))
        return
    sample = RefSample(args.config, full=args.ref_full)
    rates, secs, extra = [], [], {}
    if args.ref_throughput:
        n, w, t, b = CONFIGS[args.config]
        steps = 1
        t0 = time.perf_counter()
        procs = [subprocess.Popen([REF_DRIVER, "bench", str(sample.n), str(w), str(t), str(b), str(1000 + k), "1"],
                                  stdout=subprocess.PIPE, text=True) for k in range(cores)]
        outs = [json.loads(p.communicate()[0]) for p in procs]
        wall = time.perf_counter() - t0
        rates.append(sum(o["gflop"] for o in outs) / wall / 1e3)
        secs.append(wall)
        extra["throughput_mode"] = f"{cores} concurrent single-thread processes, one matrix each, {wall:.1f} s wall"
        workers = 1
    else:
        steps = 1 if args.ref_full else args.steps
        for _ in range(0 if args.ref_full else args.warmup):
            sample.run(cores)
        for _ in range(steps):
            r = sample.run(cores)
            rates.append(r["gflop"] / r["total_s"] / 1e3)
            secs.append(r["total_s"])
            extra = {k: r[k] for k in ("factorize_s", "phase1_s", "phase2_s", "total_s", "gflop") if k in r}
        workers = cores
        if args.ref_workers1:
            r1 = sample.run(1)
            extra["workers1"] = {"total_s": r1["total_s"], "value": r1["gflop"] / r1["total_s"] / 1e3}
    value = statistics.median(rates)
    desc = f"{sample.desc} per step ({'the full workload' if args.ref_full else 'same band/arrow/tile as the workload'}), workers={workers}"
    n = CONFIGS[args.config][0]
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world,
        "steps": steps, "warmup": args.warmup, "ms_per_step": 1e3 * statistics.median(secs),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference generator, density 1, seed 42)" if args.config != "kronecker"
        else "synthetic (Kronecker INLA precision, Matrix Market)",
        "config": {"workload": f"{args.config} (n={n}): factorize + selected inversion (pattern), reference CPU "
                               f"path on {'the full workload' if args.ref_full else 'a bounded sample'}",
                   "sample_n": sample.n, "n": n, "tile": sample.b},
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": workers, "kind": "reference",
                         "cpu_model": cpu_model(), "sample": desc},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        **({"reference_run": extra} if extra else {}),
    }), flush=True)


# ---------------------------------------------------------------------------

def relaunch_under_torchrun(args):
    """`python bench.py --gpus N` outside torchrun: one process per GPU."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="large", choices=sorted(CONFIGS))
    ap.add_argument("--batch-count", type=int, default=None, help="matrices of the batch config (default 64)")
    ap.add_argument("--tile", type=int, default=None, help="tile size b (default: the config's)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-full", action="store_true", help="reference arm: the whole workload, one run")
    ap.add_argument("--ref-workers1", action="store_true", help="reference arm: also a workers=1 run")
    ap.add_argument("--ref-throughput", action="store_true", help="reference arm: nproc concurrent 1-thread runs")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        relaunch_under_torchrun(args)
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch

    from paper_2504_19171_b200.shard import batch_seeds, max_over_ranks

    # TIB_BENCH_SAME_DEVICE=1: every rank on cuda:0 (tests on a one-GPU box)
    dev = 0 if os.environ.get("TIB_BENCH_SAME_DEVICE") == "1" else local
    torch.cuda.set_device(dev)
    dist = None
    backend = os.environ.get("TIB_BENCH_BACKEND", "nccl")
    if world > 1:
        import torch.distributed as dist

        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group(backend)
    red_dev = "cuda" if backend == "nccl" else "cpu"

    def barrier():
        if dist:
            dist.barrier()

    def mx(x):
        return max_over_ranks(x, dist, red_dev)

    import paper_2504_19171_b200 as tib

    n, w, t, b = CONFIGS[args.config]
    b = args.tile or b
    total = args.batch_count or BATCH_TOTAL.get(args.config)
    if total:
        seeds = batch_seeds(1000, total, rank, world)
        ms = [tib.generate(n, w, t, 1.0, seed=s, tile_size=b) for s in seeds]
        ms_dev = [tib.generate(n, w, t, 1.0, seed=s, tile_size=b, device=dev) for s in seeds]
    elif args.config == "kronecker":
        kc = dict(tib.KRONECKER_CONFIG)
        kc["seed"] += rank
        ms, ms_dev = [tib.generate_kronecker(tile_size=b, **kc)], None
        n = ms[0].n
    else:
        seeds = [42 + rank]
        ms = [tib.generate(n, w, t, 1.0, seed=42 + rank, tile_size=b)]
        ms_dev = [tib.generate(n, w, t, 1.0, seed=42 + rank, tile_size=b, device=dev)]
    per = len(ms)
    m = ms[0]
    flops_one = sum(tib.task_flops(m))
    flops = flops_one * per  # this rank, per step
    flops_all = flops_one * (total if total else world)  # the whole job, per step
    stored_tiles = m.stored_tiles
    h2d = stored_tiles * b * b * 8 * per
    d2h = n * 8 * per

    # ---- device-resident timing: K fused sweeps, CUDA events on the library stream
    res = tib.Resident(m if per == 1 else ms, device=dev)
    res.run(args.warmup)
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(dev) as clk:
        tot_ms, ms_fact, ms_p2 = res.run(args.steps)
        torch.cuda.synchronize()
    barrier()
    info = res.info()
    del res
    ms_step = mx(tot_ms / args.steps)
    value = flops_all / (ms_step / 1e3) / 1e12

    # ---- end to end through the public API, host buffers, H2D + D2H inside
    def public_call(mats):
        if len(mats) == 1:
            r = tib.selected_inverse(mats[0], "pattern", device=dev)
            _ = r.diagonal(), r.logdet()
            del r
        else:  # marginal variances + logdet of every matrix of the batch, one batched call
            _ = tib.selected_inverse_batch(mats, device=dev)

    def e2e_time(mats):
        public_call(mats)
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        k = max(1, min(args.steps, 3))
        for _ in range(k):
            public_call(mats)
        torch.cuda.synchronize()
        s = mx((time.perf_counter() - t0) / k)
        barrier()
        return s

    e2e_s = e2e_time(ms)
    e2e = flops_all / e2e_s / 1e12
    e2e_gen = None
    if ms_dev is not None:
        g_s = e2e_time(ms_dev)
        e2e_gen = {"value": flops_all / g_s / 1e12, "unit": "TFLOP/s", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": d2h * (total or world), "seconds_per_matrix": g_s / per,
                   "note": "generate(..., device=k): the generator runs on the GPU inside each call"}

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
    if args.config == "kronecker":
        kc = tib.KRONECKER_CONFIG
        wl = (f"kronecker AR1(rho={kc['rho']}, {kc['nt']} steps) x SPDE({kc['nx']}x{kc['ny']} lattice) + {kc['p']} "
              f"fixed effects, n={n} b={b}")
        data = "synthetic (Kronecker INLA precision, kronecker.cpp, seed 42+rank)"
    else:
        wl = f"{args.config} arrowhead n={n} w={w} t={t} b={b}"
        data = "synthetic (bit-exact reference generator, density 1, " + (
            f"seeds 1000..{999 + total} sharded over the GPUs)" if total else "seed 42+rank)")
    line = {
        "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong" if total else "weak",
        "vs_baseline": None, "dtype": "f64", "data": data,
        "config": {"workload": wl + (f" x{per} matrices per GPU (one batched launch per sweep)" if per > 1 else "")
                   + ": fused factorize + selected inversion (pattern) + marginal variances + logdet per matrix",
                   "n": n, "bandwidth": w, "thickness": t, "tile": b, "matrices_per_gpu_per_step": per,
                   "matrices_per_step": total or world,
                   "parallelism": f"independent matrices per GPU (x{world})",
                   "l2": "inputs larger than L2 (tile store %.1f GB per copy)" % (h2d / 1e9),
                   "task_model_gflop": flops_all / 1e9, "executed_gflop": info["executed_flops"] / 1e9 * (
                       (total or world) / per)},
        "seconds_per_matrix": ms_step / 1e3 / per,
        "ms_factorize_sweep": ms_fact, "ms_phase2_sweep": ms_p2,
        "logdet": info["logdet"],
        "e2e": {"value": e2e, "unit": "TFLOP/s", "h2d_bytes_per_step": h2d * (total or world) // per,
                "d2h_bytes_per_step": d2h * (total or world) // per, "seconds_per_matrix": e2e_s / per},
        "gpu_launches": int(info["kernel_launches_per_rep"]) * args.steps,
        "roofline": {"bound": "tensor", "achieved": per_gpu, "peak": peak, "unit": "TFLOP/s",
                     "frac": per_gpu / peak, "traffic": traffic, "peak_source": peak_src,
                     "kernel": "dataflow_kernel (both sweeps; task-model FLOPs / event time)"},
        "clocks": clk.summary(),
    }
    if e2e_gen:
        line["e2e_device_generated"] = e2e_gen
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args.config)
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
