"""Task-graph / complexity analyzer (csrc/dag.cpp) against the reference's
dag.cpp: reports, DOT text and closed forms equal the fixtures the reference
module wrote (tests/golden/make_golden.py dag), the known answers of
proj/tests/test_dag.cpp, and -- as a cross-check of the GPU planner -- the
phase-2 GEMM terms the device plan executes."""
import json
import os

import pytest

from conftest import GOLDEN

with open(os.path.join(GOLDEN, "dag.json")) as f:
    G = json.load(f)


def test_reports_equal_reference(tib):
    for n, b, rep in G["reports"]:
        assert tib.dag_report(n, b) == rep, (n, b)


def test_dot_text_byte_identical(tib):
    for n, b, cores, dot in G["dots"]:
        assert tib.export_dot(n, b, cores) == dot, (n, b, cores)


def test_predict_gemm_count(tib):
    for n, b, v in G["predict"]:
        assert tib.predict_gemm_count(n, b) == v
    for n in range(1, 30):  # dense closed form collapses to (N^3 - N) / 3 (test_dag.cpp:72-77)
        assert tib.predict_gemm_count(n, n) == (n ** 3 - n) // 3


def test_known_answers():
    """proj/tests/test_dag.cpp:11-59."""
    import paper_2504_19171_b200 as tib

    one = tib.dag_report(1, 1)
    assert (one["trsm"], one["lauum"], one["gemm_actual"], one["critical_path"]) == (1, 1, 0, 2)
    dense = tib.dag_report(6)
    assert (dense["trsm"], dense["trmm"], dense["lauum"], dense["gemm_actual"], dense["critical_path"]) == (6, 15, 6, 70, 32)
    assert dense["match"] and dense["gemm_predicted"] == 70
    b2 = tib.dag_report(6, 2)
    assert (b2["trmm"], b2["gemm_actual"], b2["critical_path"], b2["match"]) == (9, 26, 20, True)
    b1 = tib.dag_report(6, 1)
    assert (b1["trmm"], b1["gemm_actual"], b1["critical_path"], b1["match"]) == (5, 10, 4, True)
    b3 = tib.dag_report(6, 3)
    assert (b3["gemm_actual"], b3["critical_path"]) == (44, 26)
    # per-column increments are B^2 + B (test_dag.cpp:79-89)
    for band in (1, 2, 3, 4):
        lo, hi = tib.dag_report(band + 3, band), tib.dag_report(band + 4, band)
        assert hi["gemm_actual"] - lo["gemm_actual"] == band * band + band
    dot = tib.export_dot(1, 1)
    assert dot == 'digraph tasks {\n  rankdir=TB;\n  node [shape=box];\n  n0 [label="TRSM_INV(0,0)"];\n' \
                  '  n1 [label="LAUUM(0,0)"];\n  n0 -> n1;\n}\n'
    assert "fillcolor" not in tib.export_dot(2, 2)
    assert 'style=filled, fillcolor="#a6cee3"' in tib.export_dot(3, 2, 2)


def test_errors(tib):
    for args in [(0, 1), (3, 4)]:
        with pytest.raises(tib.TileinvError, match="tile count|band width"):
            tib.predict_gemm_count(*args)
    with pytest.raises(tib.TileinvError, match="band width"):
        tib.dag_report(4, 5)
    assert tib.export_dot(3, 2, -1) == tib.export_dot(3, 2, 0)  # cores <= 0: no assignment (module.cpp:230)


@pytest.mark.parametrize("n,w,t,b", [(20000, 2000, 200, 512), (50000, 500, 50, 128), (3000, 200, 50, 128)])
def test_graph_matches_planner_work(tib, n, w, t, b):
    """The matrix form (build_dag over the filled pattern and the pattern
    closure) counts exactly the phase-1 / phase-2 work the planner charges:
    TRSM_INV = LAUUM = N, TRMM = off-diagonal factor tiles, and the phase-2
    GEMM FLOPs 2 b^3 per node."""
    m = tib.generate(n, w, t, 1.0, seed=1, tile_size=b)
    rep = tib.dag_report_of(m)
    N = m.n_tiles
    pattern = tib.factor_pattern(m)
    assert rep["trsm"] == rep["lauum"] == N
    assert rep["trmm"] == len(pattern) - N
    _, p1, p2 = tib.task_flops(m)
    assert p2 == pytest.approx(2 * b ** 3 * rep["gemm_actual"] + N * b ** 3 / 3, rel=1e-14)
    assert p1 == pytest.approx(N * b ** 3 / 3 + rep["trmm"] * b ** 3, rel=1e-14)
