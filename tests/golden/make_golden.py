"""Regenerates the golden fixtures in tests/golden/ from the REFERENCE itself.

Run in the build container (it needs oracle/_ref, built from /root/reference by
oracle/Makefile): python tests/golden/make_golden.py.  The GPU box never runs
this; it only reads the committed fixtures.

  kat.json        known-answer cases from the reference's own tests
                  (test_smoke.py, test_selinv.cpp, test_cholesky.cpp) evaluated
                  by the reference Python module
  cases.npz       reference entries (r, c, value) for small generated cases
                  over every selection kind (test_smoke.py / acceptance-4 style)
  symbolic.json   reference factor pattern, closure, requested tiles and
                  column work lists (ref_driver symbolic) per case
  small.npz       diag(Sigma), logdet, trace of the SURVEY small config
                  (n=10000 w=200 t=50 b=128 seed 42) from ref_driver dump
  config_*.npz    BASELINE configs 2, 3, 5 (medium, large, batch members 1000
                  and 1063) from `ref_driver golden` (the reference's own
                  factorize + phase1 + phase2, 8 workers): diag(Sigma), logdet,
                  trace, payload_checksum of the generated matrix, per closure
                  tile (Frobenius norm, sum, weighted sum), and the leading /
                  trailing 64 x 64 blocks of sampled tiles (last three tile
                  columns, the middle column, arrow tiles).  Large takes ~4 min.
                  kron_small / kron_mid: config 4 (AR1 x SPDE + fixed
                  effects) at reduced scale through read_matrix_market_file
    python tests/golden/make_golden.py configs [DIR]   (DIR: reuse outputs of
    an earlier `ref_driver golden` run written as DIR/<name>.*)
  stls/*.stls.gz  tile files the reference wrote itself (`ref_driver stls`:
                  write_tile_file of the generated matrix, the factor, the
                  phase-1 tiles, and write_selected_inverse of the pattern
                  inverse) -- byte-compatibility fixtures of the STLS I/O
    python tests/golden/make_golden.py stls
  dag.json        the reference's task-graph analyzer (dag_report, export_dot,
                  predict_gemm_count of module.cpp:217-236) over small band+arrow
                  grids: reports, DOT text (plain and core-coloured), closed forms
    python tests/golden/make_golden.py dag
"""
import json
import os
import subprocess
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF = os.path.join(ROOT, "oracle", "_ref")
sys.path.insert(0, os.path.join(REF, "py"))
import tileinv as R  # noqa: E402  (the reference's pybind module)

CASES = [
    # n, w, t, density, seed, b, selection
    (24, 5, 2, 0.8, 7, 4, "all"),
    (24, 5, 2, 0.8, 7, 4, [(11, 2)]),
    (30, 4, 1, 0.9, 3, 8, "diagonal"),
    (60, 9, 3, 0.6, 11, 8, "pattern"),
    (48, 8, 3, 0.5, 23, 8, "diagonal"),
    (257, 30, 5, 0.7, 2, 32, "all"),
    (300, 40, 7, 1.0, 3, 32, "pattern"),
    (300, 40, 7, 1.0, 3, 32, [(299, 0), (150, 3), (5, 5), (200, 100), (5, 5)]),
    (500, 60, 11, 0.3, 9, 120, "pattern"),
    (700, 90, 12, 1.0, 5, 64, "diagonal"),
    (1000, 150, 20, 1.0, 13, 128, "diagonal"),
]


def sel_arg(sel):
    if isinstance(sel, str):
        return sel
    return ";".join(f"{r},{c}" for r, c in sel)


CONFIGS = {
    # name: n, w, t, b, seed
    "medium": (100000, 1000, 100, 256, 42),
    "large": (200000, 2000, 200, 512, 42),
    "batch1000": (50000, 500, 50, 128, 1000),
    "batch1063": (50000, 500, 50, 128, 1063),
}


# BASELINE config 4 at reduced scale (the reference reads these as Matrix Market
# written by this package's generator; it has no Kronecker generator of its own):
# name: nt, nx, ny, p, b  (rho 0.9, kappa2 0.5, tau 1, tau_y 1, q_beta 0.01, seed 42)
KRON = {
    "kron_small": (10, 20, 20, 20, 128),
    "kron_mid": (50, 40, 25, 20, 256),
}


def pack_config(name, prefix, info, args):
    s = info["block"]
    sampled = np.array(info["sampled"], dtype=np.int32).reshape(-1, 2)
    np.savez_compressed(
        os.path.join(HERE, f"config_{name}.npz"),
        args=np.array(args, dtype=np.int64),
        diag=np.fromfile(prefix + ".diag.f64", dtype=np.float64),
        tstats=np.fromfile(prefix + ".tstats.f64", dtype=np.float64).reshape(-1, 3),
        blocks=np.fromfile(prefix + ".blocks.f64", dtype=np.float64).reshape(len(sampled), 2, s, s),
        sampled=sampled,
        logdet=info["logdet"], trace=info["trace"],
        matrix_checksum=np.uint64(info["matrix_checksum"]),
        closure_tiles=info["closure_tiles"])


def configs(from_dir=None):
    with tempfile.TemporaryDirectory() as tmp:
        for name, args in CONFIGS.items():
            n, w, t, b, seed = args
            if from_dir:
                prefix = os.path.join(from_dir, name)
                info = json.load(open(prefix + ".json"))
            else:
                prefix = os.path.join(tmp, name)
                out = subprocess.run([os.path.join(REF, "ref_driver"), "golden", str(n), str(w), str(t), str(b),
                                      str(seed), str(os.cpu_count()), prefix],
                                     check=True, capture_output=True, text=True).stdout
                info = json.loads(out)
            pack_config(name, prefix, info, args)
            print("config", name, "logdet", info["logdet"])
        sys.path.insert(0, ROOT)
        import paper_2504_19171_b200 as tib
        for name, args in KRON.items():
            nt, nx, ny, p, b = args
            if from_dir:
                prefix = os.path.join(from_dir, name)
                info = json.load(open(prefix + ".json"))
            else:
                prefix = os.path.join(tmp, name)
                tib.write_matrix_market(tib.generate_kronecker(nt, nx, ny, p, tile_size=b), prefix + ".mtx")
                out = subprocess.run([os.path.join(REF, "ref_driver"), "golden_mm", prefix + ".mtx", str(b),
                                      str(os.cpu_count()), prefix], check=True, capture_output=True, text=True).stdout
                info = json.loads(out)
            pack_config(name, prefix, info, args)
            print("config", name, "logdet", info["logdet"])


STLS_CASES = {"case_b32": (200, 30, 6, 32, 4), "case_b100": (250, 30, 6, 100, 3)}  # n, w, t, b, seed


def stls():
    import gzip
    import shutil
    out = os.path.join(HERE, "stls")
    os.makedirs(out, exist_ok=True)
    with tempfile.TemporaryDirectory() as tmp:
        for name, (n, w, t, b, seed) in STLS_CASES.items():
            subprocess.run([os.path.join(REF, "ref_driver"), "stls", str(n), str(w), str(t), str(b), str(seed),
                            os.path.join(tmp, name)], check=True)
            for kind in ("matrix", "factor", "phase1", "sigma"):
                with open(os.path.join(tmp, f"{name}.{kind}.stls"), "rb") as fi, \
                        gzip.GzipFile(os.path.join(out, f"{name}.{kind}.stls.gz"), "wb", compresslevel=9, mtime=0) as fo:
                    shutil.copyfileobj(fi, fo)
    print("stls fixtures:", sorted(os.listdir(out)))


DAG_GRIDS = [(n, b) for n in range(1, 11) for b in range(0, n + 1)] + [(24, 3), (40, 5), (61, 7)]


def dag():
    out = {"reports": [], "dots": [], "predict": []}
    for n, b in DAG_GRIDS:
        out["reports"].append([n, b, R.dag_report(n, b)])
    for n, b in DAG_GRIDS:
        if n <= 7:
            for cores in (0, 3, 9):
                out["dots"].append([n, b, cores, R.export_dot(n, b, cores)])
    for n in (1, 2, 7, 391, 1000, 4096):
        for b in sorted({1, 2, 5, min(n, 11), n}):
            if b <= n:
                out["predict"].append([n, b, R.predict_gemm_count(n, b)])
    with open(os.path.join(HERE, "dag.json"), "w") as f:
        json.dump(out, f)


def main():
    if len(sys.argv) > 1 and sys.argv[1] == "dag":
        dag()
        return
    if len(sys.argv) > 1 and sys.argv[1] == "stls":
        stls()
        return
    if len(sys.argv) > 1 and sys.argv[1] == "configs":
        configs(sys.argv[2] if len(sys.argv) > 2 else None)
        return
    kat = {}
    a = np.array([[4.0, 2.0], [2.0, 5.0]])
    kat["two_by_two_all"] = R.selected_inverse(R.from_dense(a), "all").entries()
    kat["identity5_diag_b2"] = R.selected_inverse(R.from_dense(np.eye(5), tile_size=2), "diagonal").entries()
    kat["diag_4_2_10_half"] = R.selected_inverse(R.from_dense(np.diag([4.0, 2.0, 10.0, 0.5]), tile_size=2),
                                                 "diagonal").entries()
    try:
        R.factorize(R.from_dense(np.array([[1.0, 2.0], [2.0, 1.0]])))
    except R.NotSpdError as e:
        kat["not_spd_2x2"] = str(e)
    d = np.eye(6)
    d[4, 4] = -1.0
    try:
        R.factorize(R.from_dense(d, tile_size=2))
    except R.NotSpdError as e:
        kat["not_spd_pivot4"] = str(e)
    with open(os.path.join(HERE, "kat.json"), "w") as f:
        json.dump(kat, f, indent=1)

    arrays, sym = {}, {}
    for k, (n, w, t, dens, seed, b, sel) in enumerate(CASES):
        m = R.generate(n, w, t, dens, seed=seed, tile_size=b)
        res = R.selected_inverse(m, sel)
        ent = np.array(res.entries(), dtype=np.float64).reshape(-1, 3)
        arrays[f"case{k}"] = ent
        out = subprocess.run([os.path.join(REF, "ref_driver"), "symbolic", str(n), str(w), str(t), str(b), str(seed),
                              repr(dens), sel_arg(sel)], check=True, capture_output=True, text=True).stdout
        sym[f"case{k}"] = {"args": [n, w, t, dens, seed, b, sel if isinstance(sel, str) else [list(p) for p in sel]],
                           **json.loads(out)}
    np.savez_compressed(os.path.join(HERE, "cases.npz"), **arrays)
    with open(os.path.join(HERE, "symbolic.json"), "w") as f:
        json.dump(sym, f)

    with tempfile.TemporaryDirectory() as tmp:
        out = subprocess.run([os.path.join(REF, "ref_driver"), "dump", "10000", "200", "50", "128", "42", "8",
                              os.path.join(tmp, "small")], check=True, capture_output=True, text=True).stdout
        info = json.loads(out)
        diag = np.fromfile(os.path.join(tmp, "small.diag.f64"), dtype=np.float64)
    np.savez_compressed(os.path.join(HERE, "small.npz"), diag=diag, logdet=info["logdet"], trace=info["trace"],
                        gflop=info["gflop"], gflop_factorize=info["gflop_factorize"],
                        gflop_phase1=info["gflop_phase1"], gflop_phase2=info["gflop_phase2"])
    print("golden fixtures written:", sorted(os.listdir(HERE)))


if __name__ == "__main__":
    main()
