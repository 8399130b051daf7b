"""Device path vs the reference's golden vectors and the CPU oracle (bit-exact).

Everything here goes through the product API, which calls the sm_100a kernels
through the C ABI; the expected values come from running the reference itself
(tests/golden) or the pinned oracle.
"""
import math

import numpy as np
import pytest

import paper_1502_07451_b200 as H
from paper_1502_07451_b200 import _native, costs
from paper_1502_07451_b200.graph import CPU, GPU
from paper_1502_07451_b200.partition import (Partition, PartitionConfig, PartitionError,
                                             brute_force_partition, evaluate, fm_refine,
                                             partition_heuristic)
from paper_1502_07451_b200.policies import GraphPartitionPolicy, build_policy
from paper_1502_07451_b200.sim import (MachineModel, SimulationError, compare, compare_csv,
                                       critical_path_lower_bound, simulate, trace_csv)
from oracle import hetsched_oracle as O

from _util import bits, graph_from_spec, make_graph, random_weighted_graph

pytestmark = pytest.mark.gpu


def _all(small_cases, medium_cases):
    return small_cases + medium_cases


def _part_matches(p, rec, g, name):
    assert bits(p.assignment, g) == rec["assign"], name
    assert p.edge_cut == rec["edge_cut"], name
    assert p.balance_error == rec["balance_error"], name
    assert p.feasible == rec["feasible"], name
    assert list(p.side_weights) == rec["side_weights"], name


def test_totals_ratio_critical_path(small_cases, medium_cases):
    for c in _all(small_cases, medium_cases):
        g = graph_from_spec(c["spec"])
        assert list(H.total_weights(g)) == c["total_weights"], c["name"]
        assert H.workload_ratio(g).r_cpu == c["workload_ratio"], c["name"]
        assert critical_path_lower_bound(g) == c["critical_path"], c["name"]


def test_evaluate_bit_exact(small_cases, medium_cases):
    for c in _all(small_cases, medium_cases):
        g = graph_from_spec(c["spec"])
        ev = c["evaluate_alt"]
        ids = g.kernel_ids()
        a = {i: (CPU if ch == "0" else GPU) for i, ch in zip(ids, ev["assign"])}
        cut, err, sides = evaluate(g, Partition(a, 0.0, 0.0, H.PartitionTargets(0.5, 0.5)))
        assert (cut, err, list(sides)) == (ev["edge_cut"], ev["balance_error"],
                                           ev["side_weights"]), c["name"]


def test_partition_heuristic_bit_exact(small_cases, medium_cases):
    for c in _all(small_cases, medium_cases):
        g = graph_from_spec(c["spec"])
        half = H.PartitionTargets(0.5, 0.5)
        _part_matches(partition_heuristic(g, half), c["heuristic_half"], g, c["name"])
        t = H.workload_ratio(g)
        _part_matches(partition_heuristic(g, t), c["heuristic_ratio"], g, c["name"])
        p = partition_heuristic(g, H.PartitionTargets(0.4, 0.6),
                                PartitionConfig(imbalance_tolerance=0.25, seed=1))
        _part_matches(p, c["heuristic_loose_seed1"], g, c["name"])
        p = partition_heuristic(g, half, PartitionConfig(node_weight_source=CPU,
                                                         imbalance_tolerance=0.05))
        _part_matches(p, c["heuristic_cpu_source"], g, c["name"])


def test_fm_refine_bit_exact(small_cases, medium_cases):
    for c in _all(small_cases, medium_cases):
        g = graph_from_spec(c["spec"])
        ids = g.kernel_ids()
        ev = c["evaluate_alt"]
        a = {i: (CPU if ch == "0" else GPU) for i, ch in zip(ids, ev["assign"])}
        half = H.PartitionTargets(0.5, 0.5)
        p0 = Partition(a, ev["edge_cut"], ev["balance_error"], half)
        out = fm_refine(g, p0, half, PartitionConfig(imbalance_tolerance=0.25))
        _part_matches(out, c["fm_refine_alt"], g, c["name"])


def test_brute_force_bit_exact(small_cases):
    for c in small_cases:
        if "brute_half" not in c:
            continue
        g = graph_from_spec(c["spec"])
        p = brute_force_partition(g, H.PartitionTargets(0.5, 0.5), 0.25)
        _part_matches(p, c["brute_half"], g, c["name"])


def test_simulate_bit_exact(small_cases, medium_cases):
    for c in _all(small_cases, medium_cases):
        g = graph_from_spec(c["spec"])
        for key, rec in c["simulate"].items():
            pol, cw, gw = key.split("_")
            tr = simulate(g, build_policy(pol, g), MachineModel(int(cw), int(gw)))
            assert tr.makespan == rec["makespan"], (c["name"], key)
            assert tr.transfer_count == rec["transfer_count"], (c["name"], key)
            assert tr.transfer_bytes == rec["transfer_bytes"], (c["name"], key)
            assert [tr.busy_ms[CPU], tr.busy_ms[GPU]] == rec["busy"], (c["name"], key)
            assert [tr.kernels_per_device[CPU], tr.kernels_per_device[GPU]] == rec["kpd"]
            import hashlib
            assert hashlib.sha256(trace_csv(tr).encode()).hexdigest() == rec["trace_sha256"], \
                (c["name"], key)


def test_compare_matches_reference(compare_golden):
    factory = lambda s: H.attach_weights(  # noqa: E731
        H.generate_random_dag(38, 75, "MA", 1024, seed=s), costs.SyntheticCostModel())
    rows = compare(["eager", "dmda", "gp"], factory, MachineModel(3, 1),
                   iterations=compare_golden["iterations"], seed=compare_golden["seed"])
    for r, g in zip(rows, compare_golden["rows"]):
        for k, v in g.items():
            assert getattr(r, k) == v, (r.policy, k)
    assert compare_csv(rows) == compare_golden["csv"]


def test_known_answers():
    """The reference's hand-derived tests (test_partition.py:76-104, test_sim.py:53-153)."""
    g = make_graph({1: (1.0, 1.0), 2: (1.0, 1.0), 3: (1.0, 1.0)}, [(1, 2, 5.0), (2, 3, 1.0)])
    p = brute_force_partition(g, H.PartitionTargets(1.0 / 3.0, 2.0 / 3.0), tolerance=0.05)
    assert p.assignment == {1: GPU, 2: GPU, 3: CPU} and p.edge_cut == 1.0 and p.feasible
    g = make_graph({1: (1.0, 1.0), 2: (100.0, 100.0)}, [])
    p = brute_force_partition(g, H.PartitionTargets(0.5, 0.5), tolerance=0.01)
    assert not p.feasible and p.balance_error == pytest.approx(abs(1 / 101 - 0.5))
    big = make_graph({i: (1.0, 1.0) for i in range(1, 22)}, [])
    with pytest.raises(PartitionError, match="limit 20"):
        brute_force_partition(big, H.PartitionTargets(0.5, 0.5), 0.1)
    g = make_graph({1: (1.0, 1.0), 2: (1.0, 1.0), 3: (1.0, 1.0), 4: (1.0, 1.0)},
                   [(1, 2, 5.0), (3, 4, 5.0), (2, 3, 0.1)])
    p = partition_heuristic(g, H.PartitionTargets(0.5, 0.5),
                            PartitionConfig(imbalance_tolerance=0.05))
    assert p.edge_cut == pytest.approx(0.1) and p.feasible
    g = make_graph({1: (5.0, 9.0)}, [])
    tr = simulate(g, H.build_policy("eager", g))
    assert tr.makespan == 5.0 and tr.transfer_count == 0
    assert tr.kernels_per_device == {CPU: 1, GPU: 0}
    g = make_graph({1: (2.0, 9.0), 2: (2.0, 9.0), 3: (9.0, 1.0)}, [(1, 3, 2.0), (2, 3, 2.0)])
    tr = simulate(g, GraphPartitionPolicy({1: CPU, 2: CPU, 3: GPU}))
    assert tr.makespan == 7.0 and tr.transfer_count == 2
    g = make_graph({1: (9.0, 1.0), 2: (9.0, 1.0)}, [(1, 2, 5.0)])
    tr = simulate(g, GraphPartitionPolicy({1: GPU, 2: GPU}))
    assert [e.subject for e in tr.events if e.kind == "xfer_start"] == ["d0.1"]
    assert tr.makespan == 2.0
    g = make_graph({1: (2.0, 5.0), 2: (2.0, 5.0)}, [(1, 2, 1.0)])
    assert critical_path_lower_bound(g) == 4.0
    g = make_graph({1: (1.0, 9.0), 2: (7.0, 9.0)}, [])
    assert critical_path_lower_bound(g) == 7.0
    g = random_weighted_graph(9)
    tr = simulate(g, H.build_policy("eager", g), MachineModel(1, 0))
    assert tr.makespan == pytest.approx(sum(g.nodes[i].weight_cpu for i in g.kernel_ids()))


def test_error_conventions():
    from paper_1502_07451_b200.graph import KernelNode, ROOT_ID, SOURCE_KIND, TaskGraph
    g = TaskGraph([KernelNode(ROOT_ID, SOURCE_KIND, 0), KernelNode(1, "K", 8, 1.0, 1.0)], [])
    with pytest.raises(SimulationError, match="invalid graph"):
        simulate(g, H.build_policy("eager", g))
    g = make_graph({1: (0.0, 0.0)}, [])
    with pytest.raises(SimulationError, match="cost model"):
        simulate(g, H.build_policy("eager", g))
    with pytest.raises(PartitionError):
        partition_heuristic(g, H.PartitionTargets(0.5, 0.5))

    class Custom:
        name = "custom"
    g = make_graph({1: (1.0, 1.0)}, [])
    with pytest.raises(SimulationError, match="native backend"):
        simulate(g, Custom())


def test_random_graphs_against_oracle():
    """Fresh seeded graphs beyond the fixtures: device == oracle, bit for bit."""
    for seed in range(200, 260):
        g = random_weighted_graph(seed, max_kernels=20)
        from _util import spec_of
        og = O.OGraph(spec_of(g))
        r = H.workload_ratio(g).r_cpu
        assert r == O.workload_ratio(og)
        p = partition_heuristic(g, H.workload_ratio(g))
        assert bits(p.assignment, g) == bits(O.partition_heuristic(og, r), g)
        for pol in ("eager", "dmda", "gp"):
            pin = p.assignment if pol == "gp" else None
            tr = simulate(g, GraphPartitionPolicy(pin) if pin else H.build_policy(pol, g))
            ref = O.simulate(og, pol, pin)
            assert tr.makespan == ref["makespan"] and tr.transfer_count == ref["transfer_count"]


def test_batched_partition_equals_single():
    from paper_1502_07451_b200.partition import partition_heuristic_batch
    from paper_1502_07451_b200.costs import workload_ratio_batch
    graphs = [random_weighted_graph(s, max_kernels=18) for s in range(300, 340)]
    targets = workload_ratio_batch(graphs)
    assert [t.r_cpu for t in targets] == [H.workload_ratio(g).r_cpu for g in graphs]
    batch = partition_heuristic_batch(graphs, targets)
    for g, t, a in zip(graphs, targets, batch):
        assert a == partition_heuristic(g, t).assignment
