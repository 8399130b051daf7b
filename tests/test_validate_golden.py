"""validate / topological_order against the REFERENCE's own outputs.

tests/golden/validate.json was produced by running the unmodified reference
(graph.py:113-172) on the graphs of tests/_validate_cases.py
(tests/golden/make_validate_golden.py): crafted invalid graphs (self-loops,
cycles, negative weights, weighted roots, kernels without predecessors, a
root that is not the smallest id, sparse id ranges) and seeded random DAGs
with arbitrary numbering, some closed into cycles.

CPU: the oracle's restatement reproduces every golden order / cycle member.
GPU: the drop-in's validate() reproduces every message list; the device
validation (hs_validate_dag) reproduces the CSR-checkable messages; the device
topological_order (hs_topological_order) reproduces every order and raises
the reference's CycleError member — and, at 100k tasks / 1M edges, equals the
oracle's heap order both for creation-order numbering (identity fast path)
and for a random relabelling (batched heap rounds).
"""
import json
import os
import random

import pytest

import _validate_cases as VC
from oracle import hetsched_oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))
with open(os.path.join(HERE, "golden", "validate.json")) as f:
    GOLD = json.load(f)["cases"]
HOST_ONLY = ("duplicate node", "duplicate edge", "references unknown", "is not kind", "missing")


def test_cases_match_golden_specs():
    assert [(n, s) for n, s in VC.cases()] == [(c["name"], c["spec"]) for c in GOLD]


def test_oracle_topological_order_matches_reference():
    for c in GOLD:
        g = O.OGraph(c["spec"])
        if "cycle_member" in c:
            with pytest.raises(ValueError, match=f"node {c['cycle_member']}$"):
                O.topological_order(g)
        else:
            assert O.topological_order(g) == c["topological_order"], c["name"]


@pytest.mark.gpu
def test_validate_messages_match_reference():
    from _util import graph_from_spec
    from paper_1502_07451_b200.csr import DagCSR
    from paper_1502_07451_b200.graph import validate
    for c in GOLD:
        g = graph_from_spec(c["spec"])
        assert validate(g) == c["validate"], c["name"]
        dev = DagCSR.from_taskgraph(g).validate()
        assert dev == [m for m in c["validate"] if not any(h in m for h in HOST_ONLY)], c["name"]


@pytest.mark.gpu
def test_topological_order_matches_reference():
    from _util import graph_from_spec
    from paper_1502_07451_b200.graph import CycleError, topological_order
    for c in GOLD:
        g = graph_from_spec(c["spec"])
        if "cycle_member" in c:
            with pytest.raises(CycleError) as ei:
                topological_order(g)
            assert ei.value.member == c["cycle_member"], c["name"]
        else:
            assert topological_order(g) == c["topological_order"], c["name"]


def _layered_spec(n, m, seed, relabel):
    """A layered DAG (oracle/layered_oracle.py family) as a spec, optionally
    with the node ids randomly permuted (edges preserved)."""
    from oracle import layered_oracle
    _, edges, _ = layered_oracle.generate(n, m, seed)
    ids = list(range(n + 1))
    if relabel:
        rng = random.Random(seed)
        tail = ids[1:]
        rng.shuffle(tail)
        ids = [0] + tail
    nodes = [[ids[i], "SOURCE" if i == 0 else "MA", 0 if i == 0 else 512, 0.0, 0.0 if i == 0 else 1.0]
             for i in range(n + 1)]
    return {"root": 0, "nodes": nodes, "edges": [[ids[u], ids[v], 8, 0.1] for u, v in edges]}


@pytest.mark.gpu
@pytest.mark.parametrize("relabel", [False, True])
def test_topological_order_100k_matches_oracle(relabel):
    import numpy as np
    import torch
    from paper_1502_07451_b200 import _native
    from paper_1502_07451_b200.csr import DagCSR, HostDag
    spec = _layered_spec(100_000, 1_000_000, seed=5, relabel=relabel)
    want = O.topological_order(O.OGraph(spec))
    ids = np.array(sorted(r[0] for r in spec["nodes"]), dtype=np.int64)
    e = np.array(sorted((u, v) for u, v, _, _ in spec["edges"]), dtype=np.int64)
    h = HostDag(ids, 0, e[:, 0].astype(np.int32), e[:, 1].astype(np.int32),
                np.zeros(len(ids)), np.ones(len(ids)), np.full(len(e), 0.1),
                np.full(len(e), 8, dtype=np.int64))
    csr = DagCSR.from_host(h)
    order, count, stuck, rounds = _native.topological_order(csr)
    torch.cuda.synchronize()
    assert count == csr.n and stuck == -1
    assert (rounds == 0) == (not relabel)
    assert ids[order.cpu().numpy()].tolist() == want
