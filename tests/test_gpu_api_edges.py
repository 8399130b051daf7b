"""Edge cases of the drop-in boundary: worker counts past any fixed table, incomplete
pin maps, out-of-range k-way part ids, graphs without a root node."""
import pytest
import torch

import paper_1502_07451_b200 as H
from paper_1502_07451_b200 import kway
from paper_1502_07451_b200.graph import CPU, GPU, ROOT_ID, DataEdge, KernelNode, TaskGraph
from paper_1502_07451_b200.policies import GraphPartitionPolicy, build_policy
from paper_1502_07451_b200.sim import (MachineModel, critical_path_lower_bound, simulate,
                                       trace_csv)
from oracle import hetsched_oracle as O

from _util import random_weighted_graph, spec_of

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("cpu,gpu", [(100, 3), (70, 0), (0, 65), (5, 200)])
def test_many_workers_match_oracle(cpu, gpu):
    # the reference accepts any worker count (sim.py:27-46); the device keeps
    # per-worker state in scratch, not in a fixed table
    for seed in (3, 8):
        g = random_weighted_graph(seed, max_kernels=40)
        og = O.OGraph(spec_of(g))
        for name in ("eager", "dmda"):
            tr = simulate(g, build_policy(name, g), MachineModel(cpu, gpu))
            ref = O.simulate(og, name, None, cpu, gpu)
            assert tr.makespan == ref["makespan"], (name, seed)
            assert tr.transfer_count == ref["transfer_count"], (name, seed)


def test_incomplete_pin_map_raises_keyerror():
    # policies.py:92-93: on_ready indexes the pin map -> KeyError for a missing kernel
    g = random_weighted_graph(5, max_kernels=12)
    ids = g.kernel_ids()
    pm = {i: GPU for i in ids[1:]}
    with pytest.raises(KeyError):
        simulate(g, GraphPartitionPolicy(pm))
    pm[ids[0]] = CPU  # complete map runs
    tr = simulate(g, GraphPartitionPolicy(pm))
    assert tr.kernels_per_device[CPU] == 1


def test_evaluate_batch_rejects_out_of_range_parts():
    csr = kway.layered_dag(2000, 20000, seed=3)
    good = torch.randint(0, 8, (2, csr.n), dtype=torch.int32, device=csr.device)
    good[:, 0] = 0
    ev = kway.evaluate_batch(csr, good, 8)
    assert (ev["cut_edges"] >= 0).all()
    bad = good.clone()
    bad[1, 17] = 8
    with pytest.raises(ValueError, match="outside"):
        kway.evaluate_batch(csr, bad, 8)
    ev = kway.evaluate_batch(csr, bad, 8, check=False)
    assert ev["cut_edges"][1].item() == -1 and ev["cut_edges"][0].item() >= 0
    bad[1, 17] = -1
    with pytest.raises(ValueError):
        kway.evaluate_batch(csr, bad, 8)


def test_rootless_graph_totals_ratio_critical_path():
    # graph.py:327-332, costs.py:239-253 and sim.py:239-247 never touch the root
    nodes = [KernelNode(i, "K", 64, weight_cpu=float(i), weight_gpu=0.5 * i) for i in (1, 2, 3, 4)]
    edges = [DataEdge(1, 2, 8, 0.25), DataEdge(2, 4, 8, 0.5), DataEdge(3, 4, 8, 0.125)]
    g = TaskGraph(nodes, edges, root=ROOT_ID)
    assert ROOT_ID not in g.nodes
    og = O.OGraph(spec_of(g))
    assert list(H.total_weights(g)) == list(O.total_weights(og))
    assert H.workload_ratio(g).r_cpu == O.workload_ratio(og)
    assert critical_path_lower_bound(g) == O.critical_path(og)


def test_trace_with_many_workers_is_sorted_and_complete():
    g = random_weighted_graph(11, max_kernels=30)
    tr = simulate(g, build_policy("eager", g), MachineModel(80, 2))
    starts = [e for e in tr.events if e.kind == "kernel_start"]
    assert len(starts) == len(g.kernel_ids())
    assert trace_csv(tr).count("\n") == len(tr.events) + 1
