"""METIS wire boundary on the device vs the reference (tests/golden/metis_io.json,
made by tests/golden/make_metis_golden.py from the unmodified reference)."""
import json
import os

import numpy as np
import pytest
import torch

from paper_1502_07451_b200 import graphio, kway
from paper_1502_07451_b200.costs import workload_ratio
from paper_1502_07451_b200.partition import PartitionError
from _util import graph_from_spec  # noqa: E402

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "metis_io.json")


@pytest.fixture(scope="module")
def golden():
    with open(GOLDEN) as f:
        return json.load(f)


def test_emit_metis_matches_reference(golden):
    for rec in golden["graphs"]:
        g = graph_from_spec(rec["spec"])
        assert graphio.emit_metis(g, "GPU") == rec["metis_GPU"]
        assert graphio.emit_metis(g, "CPU") == rec["metis_CPU"]
        assert graphio.emit_metis(g, "GPU", scale=7) == rec["metis_scale7"]


def test_emit_metis_zero_weights_error(golden):
    from paper_1502_07451_b200.graph import DataEdge, KernelNode, ROOT_ID, SOURCE_KIND, TaskGraph
    ns = [KernelNode(ROOT_ID, SOURCE_KIND, 0), KernelNode(1, "K", 64), KernelNode(2, "K", 64)]
    zero = TaskGraph(ns, [DataEdge(0, 1), DataEdge(1, 2, bytes=0, weight_xfer=0.0)])
    with pytest.raises(PartitionError) as exc:
        graphio.emit_metis(zero)
    assert str(exc.value) == golden["zero_weights_error"]


def test_parse_partition_file_matches_reference(golden):
    g = graph_from_spec(golden["partition_graph"])
    t = workload_ratio(g)
    for rec in golden["partition_files"]:
        if "error" in rec:
            with pytest.raises(PartitionError) as exc:
                graphio.parse_partition_file(rec["text"], g, t)
            assert str(exc.value) == rec["error"], rec["name"]
        else:
            p = graphio.parse_partition_file(rec["text"], g, t)
            assert [p.assignment[k] for k in g.kernel_ids()] == rec["assignment"], rec["name"]
            assert p.edge_cut == rec["edge_cut"] and p.balance_error == rec["balance_error"]
            assert graphio.parse_partition_file(graphio.emit_partition_file(p, g), g, t).assignment \
                == p.assignment


def test_config2_round_trip_and_rows():
    """100k/1M: the emitted text parses back to the graph's rows; a partition file round-trips."""
    csr = kway.layered_dag(100_000, 1_000_000, seed=2)
    text = graphio.emit_metis_csr(csr)
    data = bytes(text.cpu().numpy())
    lines = data.split(b"\n")
    assert lines[-1] == b""
    n, m, fmt = lines[0].split()
    assert (int(n), fmt) == (csr.n - 1, b"011")
    ug = kway.symmetrize(csr)
    assert int(m) * 2 == ug.nnz
    xadj = ug.xadj.cpu().numpy()
    adj, w = ug.adjncy.cpu().numpy(), ug.adjwgt.cpu().numpy()
    vw = ug.vwgt.cpu().numpy()
    rng = np.random.default_rng(0)
    for v in rng.integers(0, ug.n, 200):
        toks = list(map(int, lines[1 + v].split()))
        assert toks[0] == vw[v]
        row = sorted(zip(adj[xadj[v]:xadj[v + 1]] + 1, w[xadj[v]:xadj[v + 1]]))
        assert list(zip(toks[1::2], toks[2::2])) == [(int(a), int(b)) for a, b in row]
    part = (torch.arange(ug.n, device="cuda") % 2).to(torch.int8)
    back, err = graphio.parse_partition_bytes(graphio.emit_partition_bytes(part).cpu().numpy()
                                              .tobytes(), ug.n)
    assert err is None and torch.equal(back, part)


def test_config4_partition_file_round_trip():
    """10M lines through the device parser."""
    n = 10_000_000
    part = (torch.randint(0, 2, (n,), device="cuda", generator=None)).to(torch.int8)
    data = graphio.emit_partition_bytes(part).cpu().numpy().tobytes()
    back, err = graphio.parse_partition_bytes(data, n)
    assert err is None and torch.equal(back, part)
    bad = bytearray(data)
    bad[2 * 1234567] = ord("7")
    back, err = graphio.parse_partition_bytes(bytes(bad), n)
    assert back is None and err == "line 1234568: group must be 0 or 1, got 7"
