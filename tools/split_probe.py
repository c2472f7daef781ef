"""Upper bound of a two-chain split of the large config: the factor / phase-2
sweep times of one n=200k matrix against a batch of two n=100k halves (two
independent chains in one launch), device resident."""
import json
import sys

sys.path.insert(0, ".")
import paper_2504_19171_b200 as tib  # noqa: E402

for label, n, cnt in (("one n=200k", 200000, 1), ("two n=100k", 100000, 2), ("four n=50k", 50000, 4)):
    ms = [tib.generate(n, 2000, 200, 1.0, seed=42 + k, tile_size=512, device=0) for k in range(cnt)]
    r = tib.Resident(ms if cnt > 1 else ms[0], device=0)
    r.run(2)
    tot, f, p = r.run(3)
    print(json.dumps({"case": label, "ms_step": tot / 3, "ms_factor": f, "ms_phase2": p, "info": r.info()}), flush=True)
    del r
