"""Upper bound of a split of the large config into independent chains: the
factor / phase-2 sweep times of one n=200k matrix against batches of two and
four independent pieces (one chain each, one launch), device resident.
Reserved critical workers come from TIB_CRIT_WORKERS_FACTOR (read per plan:
run each setting in its own process)."""
import json
import sys

sys.path.insert(0, ".")
import paper_2504_19171_b200 as tib  # noqa: E402

cases = {"1": (200000, 1), "2": (100200, 2), "4": (50000, 4)}
for key in (sys.argv[1:] or ["1", "2", "4"]):
    n, cnt = cases[key]
    ms = [tib.generate(n, 2000, 200, 1.0, seed=42 + k, tile_size=512, device=0) for k in range(cnt)]
    r = tib.Resident(ms if cnt > 1 else ms[0], device=0)
    r.run(2)
    tot, f, p = r.run(3)
    print(json.dumps({"case": f"{cnt} x n={n}", "ms_step": tot / 3, "ms_factor": f, "ms_phase2": p,
                      "gflop": r.info()["task_model_flops"] / 1e9}), flush=True)
    del r
