"""The CPU reference arm synthesises its config-5 graphs on the host only
(bench._cfg5_spec: host generator + scalar SyntheticCostModel, as
attach_weights applies it, graph.py:308-324). Pinned against the graph the
unmodified reference built for seed 0 (tests/golden/medium_graphs.json);
runs without a GPU, so a device call on that arm fails here."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def test_cfg5_spec_matches_reference_graph(medium_cases):
    import bench
    gold = next(c for c in medium_cases if c["name"] == "gen_38_75_MA")["spec"]
    got = bench._cfg5_spec(0)
    assert got["root"] == gold["root"]
    assert sorted(map(list, got["nodes"])) == sorted(map(list, gold["nodes"]))
    assert sorted(map(list, got["edges"])) == sorted(map(list, gold["edges"]))
