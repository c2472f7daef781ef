"""bench.py as the driver runs it, N > 1: `--gpus 2` without a torchrun
environment re-launches itself under torch.distributed.run, the batch is
sharded by shard.batch_seeds, and rank 0 prints one line for the whole job.
On a one-GPU box both ranks share cuda:0 (TIB_BENCH_SAME_DEVICE=1) and the
host-side plumbing uses gloo (TIB_BENCH_BACKEND=gloo; no data-path
collective exists)."""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def run_bench(*extra, env_extra=None):
    env = dict(os.environ, TIB_BENCH_SAME_DEVICE="1", TIB_BENCH_BACKEND="gloo", **(env_extra or {}))
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *extra], capture_output=True, text=True,
                         env=env, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_two_ranks_batch():
    line = run_bench("--gpus", "2", "--config", "batch", "--batch-count", "9", "--steps", "1", "--warmup", "1",
                     "--no-cpu-baseline")
    assert line["n_gpus"] == 2
    assert line["config"]["matrices_per_step"] == 9
    assert line["config"]["matrices_per_gpu_per_step"] == 5  # rank 0 of an uneven 5 / 4 split
    assert line["scaling"] == "strong"
    assert line["value"] > 0 and line["e2e"]["value"] > 0


def test_two_ranks_single_matrix():
    line = run_bench("--gpus", "2", "--config", "small", "--steps", "1", "--warmup", "1", "--no-cpu-baseline")
    assert line["n_gpus"] == 2 and line["scaling"] == "weak"
    assert line["config"]["matrices_per_step"] == 2
