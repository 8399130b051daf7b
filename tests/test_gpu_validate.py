"""Device validation (hs_validate_dag) against the host restatement of validate (graph.py:113-150).

Same messages in the same order for every CSR-checkable violation: negative
node weights, non-zero root weights, self-loops, negative transfer weights and
byte counts, cycles (the reference's CycleError member: the smallest id never
released by Kahn's algorithm), kernels without predecessors.
"""
import pytest
import torch

from paper_1502_07451_b200 import kway
from paper_1502_07451_b200.csr import DagCSR
from paper_1502_07451_b200.graph import (ROOT_ID, SOURCE_KIND, DataEdge, KernelNode, TaskGraph,
                                         validate)
from _util import graph_from_spec, random_weighted_graph  # noqa: E402

pytestmark = pytest.mark.gpu

HOST_ONLY = ("duplicate node", "duplicate edge", "references unknown", "is not kind", "missing")


def host_csr_messages(g):
    return [m for m in validate(g) if not any(h in m for h in HOST_ONLY)]


def _graph(nodes, edges):
    ns = [KernelNode(ROOT_ID, SOURCE_KIND, 0)] + [KernelNode(i, "K", 64, weight_cpu=wc,
                                                             weight_gpu=wg)
                                                  for i, wc, wg in nodes]
    return TaskGraph(ns, [DataEdge(u, v, bytes=b, weight_xfer=w) for u, v, b, w in edges])


CASES = {
    "valid_chain": ([(1, 1.0, 1.0), (2, 1.0, 1.0)], [(0, 1, 0, 0.0), (1, 2, 8, 0.5)]),
    "self_loop": ([(1, 1.0, 1.0), (2, 1.0, 1.0)], [(0, 1, 0, 0.0), (1, 2, 8, 0.5), (2, 2, 8, 0.5)]),
    "cycle": ([(1, 1.0, 1.0), (2, 1.0, 1.0), (3, 1.0, 1.0), (4, 1.0, 1.0)],
              [(0, 1, 0, 0.0), (1, 2, 8, 0.5), (2, 3, 8, 0.5), (3, 2, 8, 0.5), (3, 4, 8, 0.5)]),
    "negative": ([(1, -1.0, 1.0), (2, 1.0, -2.0)], [(0, 1, 0, 0.0), (1, 2, -8, -0.5)]),
    "no_root_edge": ([(1, 1.0, 1.0), (2, 1.0, 1.0), (3, 1.0, 1.0)], [(0, 1, 0, 0.0)]),
    "many": ([(1, -1.0, 1.0), (2, 1.0, 1.0), (3, 1.0, 1.0)],
             [(1, 1, 0, -1.0), (1, 2, 8, 0.5), (2, 1, 8, 0.5), (3, 3, -1, 0.1)]),
}


@pytest.mark.parametrize("name", sorted(CASES))
def test_crafted_graphs_match_host_messages(name):
    g = _graph(*CASES[name])
    dev = DagCSR.from_taskgraph(g).validate()
    assert dev == host_csr_messages(g), (dev, validate(g))
    assert (dev == []) == (name == "valid_chain")


def test_root_with_weight():
    ns = [KernelNode(ROOT_ID, SOURCE_KIND, 0, weight_cpu=1.0), KernelNode(1, "K", 64, 1.0, 1.0)]
    g = TaskGraph(ns, [DataEdge(0, 1)])
    assert DagCSR.from_taskgraph(g).validate() == host_csr_messages(g) != []


def test_golden_and_random_graphs_are_valid(small_cases):
    for case in small_cases[:20]:
        g = graph_from_spec(case["spec"])
        assert DagCSR.from_taskgraph(g).validate() == host_csr_messages(g) == []
    for seed in range(10):
        g = random_weighted_graph(seed, max_kernels=40)
        assert DagCSR.from_taskgraph(g).validate() == []


def test_random_cycles_report_the_reference_member():
    import random
    for seed in range(12):
        g = random_weighted_graph(seed + 100, max_kernels=30)
        rng = random.Random(seed)
        ks = sorted(g.kernel_ids())
        a, b = sorted(rng.sample(ks, 2))
        # a back edge b -> a closes a cycle whenever a reaches b
        edges = list(g.edges.values()) + [DataEdge(b, a, bytes=4, weight_xfer=0.1)]
        g2 = TaskGraph(list(g.nodes.values()), edges)
        assert DagCSR.from_taskgraph(g2).validate() == host_csr_messages(g2)


def test_config4_dag_is_valid():
    csr = kway.layered_dag(10_000_000, 100_000_000, seed=0)
    torch.cuda.synchronize()
    assert csr.validate() == []
