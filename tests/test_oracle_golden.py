"""Pins the CPU oracle (oracle/hetsched_oracle.py) to the reference's own outputs.

The golden vectors were produced by running the reference package itself
(tests/golden/make_golden.py); every oracle function must reproduce them
exactly (integers, assignments, fp64 bits).
"""
import math

import pytest

from oracle import hetsched_oracle as O

CPU, GPU = "CPU", "GPU"


def _bits(a, g):
    return "".join("0" if a[i] == CPU else "1" for i in g.kernel_ids())


def _cases(small_cases, medium_cases):
    return small_cases + medium_cases


def test_graph_quantities(small_cases, medium_cases):
    for c in _cases(small_cases, medium_cases):
        g = O.OGraph(c["spec"])
        assert O.topological_order(g) == c["topological_order"], c["name"]
        assert list(O.total_weights(g)) == c["total_weights"], c["name"]
        assert O.workload_ratio(g) == c["workload_ratio"], c["name"]
        assert O.critical_path(g) == c["critical_path"], c["name"]


def test_evaluate_and_fm(small_cases, medium_cases):
    for c in _cases(small_cases, medium_cases):
        g = O.OGraph(c["spec"])
        ids = g.kernel_ids()
        ev = c["evaluate_alt"]
        alt = {i: (CPU if ch == "0" else GPU) for i, ch in zip(ids, ev["assign"])}
        cut, err, sides = O.evaluate(g, alt, 0.5)
        assert (cut, err, list(sides)) == (ev["edge_cut"], ev["balance_error"],
                                           ev["side_weights"]), c["name"]
        out = O.fm_refine(g, alt, 0.5, 0.25)
        assert _bits(out, g) == c["fm_refine_alt"]["assign"], c["name"]


def test_heuristic(small_cases):
    for c in small_cases:
        g = O.OGraph(c["spec"])
        a = O.partition_heuristic(g, 0.5)
        assert _bits(a, g) == c["heuristic_half"]["assign"], c["name"]
        a = O.partition_heuristic(g, c["workload_ratio"])
        assert _bits(a, g) == c["heuristic_ratio"]["assign"], c["name"]
        a = O.partition_heuristic(g, 0.4, tol=0.25, seed=1)
        assert _bits(a, g) == c["heuristic_loose_seed1"]["assign"], c["name"]
        a = O.partition_heuristic(g, 0.5, tol=0.05, source=CPU)
        assert _bits(a, g) == c["heuristic_cpu_source"]["assign"], c["name"]


def test_heuristic_medium(medium_cases):
    for c in medium_cases[:3]:
        g = O.OGraph(c["spec"])
        a = O.partition_heuristic(g, c["workload_ratio"])
        assert _bits(a, g) == c["heuristic_ratio"]["assign"], c["name"]


def test_brute_force(small_cases):
    for c in small_cases:
        if "brute_half" not in c:
            continue
        g = O.OGraph(c["spec"])
        a = O.brute_force(g, 0.5, 0.25)
        assert _bits(a, g) == c["brute_half"]["assign"], c["name"]


def test_simulate(small_cases, medium_cases):
    for c in _cases(small_cases, medium_cases):
        g = O.OGraph(c["spec"])
        for key, rec in c["simulate"].items():
            pol, cw, gw = key.split("_")
            pin = None
            if pol == "gp":
                hr = c["heuristic_ratio"]["assign"]
                pin = {i: (CPU if ch == "0" else GPU) for i, ch in zip(g.kernel_ids(), hr)}
            r = O.simulate(g, pol, pin, int(cw), int(gw))
            assert r["makespan"] == rec["makespan"], (c["name"], key)
            assert r["transfer_count"] == rec["transfer_count"], (c["name"], key)
            assert r["transfer_bytes"] == rec["transfer_bytes"], (c["name"], key)
            assert [r["busy_ms"][CPU], r["busy_ms"][GPU]] == rec["busy"], (c["name"], key)
            assert [r["kernels_per_device"][CPU], r["kernels_per_device"][GPU]] == rec["kpd"]
            if rec["trace_csv"] is not None:
                lines = ["time,kind,subject,resource"] + [
                    f"{t!r},{k},{s},{res}" for (t, k, s, res) in r["events"]]
                assert "\n".join(lines) + "\n" == rec["trace_csv"], (c["name"], key)


def test_known_answers():
    """The reference's hand-derived cases (pkg/tests/test_partition.py:76-104,
    test_sim.py:53-85, test_sim.py:146-153)."""
    def mk(nw, edges):
        nodes = [[0, "SOURCE", 0, 0.0, 0.0]] + [[i, "K", 64, a, b] for i, (a, b) in nw.items()]
        es = [[u, v, 0, w] for (u, v, w) in edges]
        have = {v for (_, v, _) in edges}
        es += [[0, i, 0, 0.0] for i in nw if i not in have]
        return O.OGraph({"root": 0, "nodes": nodes, "edges": es})

    g = mk({1: (1.0, 1.0), 2: (1.0, 1.0), 3: (1.0, 1.0)}, [(1, 2, 5.0), (2, 3, 1.0)])
    a = O.brute_force(g, 1.0 / 3.0, 0.05)
    assert a == {1: GPU, 2: GPU, 3: CPU}
    assert O.evaluate(g, a, 1.0 / 3.0)[0] == 1.0
    g = mk({1: (1.0, 1.0), 2: (100.0, 100.0)}, [])
    a = O.brute_force(g, 0.5, 0.01)
    assert math.isclose(O.evaluate(g, a, 0.5)[1], abs(1 / 101 - 0.5))
    g = mk({1: (2.0, 9.0), 2: (2.0, 9.0), 3: (9.0, 1.0)}, [(1, 3, 2.0), (2, 3, 2.0)])
    r = O.simulate(g, "gp", {1: CPU, 2: CPU, 3: GPU})
    assert r["makespan"] == 7.0 and r["transfer_count"] == 2
    g = mk({1: (2.0, 5.0), 2: (2.0, 5.0)}, [(1, 2, 1.0)])
    assert O.critical_path(g) == 4.0


def test_oracle_metis_io_matches_reference_golden():
    """The oracle's METIS restatement against the reference's own outputs."""
    import json
    import os
    with open(os.path.join(os.path.dirname(__file__), "golden", "metis_io.json")) as f:
        gold = json.load(f)
    for rec in gold["graphs"]:
        og = O.OGraph(rec["spec"])
        assert O.emit_metis(og, "GPU") == rec["metis_GPU"]
        assert O.emit_metis(og, "CPU") == rec["metis_CPU"]
        assert O.emit_metis(og, "GPU", scale=7) == rec["metis_scale7"]
    og = O.OGraph(gold["partition_graph"])
    n = len(og.kernel_ids())
    for rec in gold["partition_files"]:
        if "error" in rec:
            try:
                O.parse_partition_groups(rec["text"], n)
                raise AssertionError(rec["name"])
            except ValueError as exc:
                assert str(exc) == rec["error"]
        else:
            got = O.parse_partition_groups(rec["text"], n)
            assert ["CPU" if v == 0 else "GPU" for v in got] == rec["assignment"]
