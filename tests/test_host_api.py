"""Host-side mirror of the reference interface: object model, generators,
cost models, validation and error conventions (no GPU needed)."""
import pytest

from paper_1502_07451_b200 import costs, gen
from paper_1502_07451_b200.graph import (CycleError, DataEdge, KernelNode, TaskGraph,
                                         topological_order, validate)
from paper_1502_07451_b200.partition import PartitionConfig, PartitionError
from paper_1502_07451_b200.sim import MachineModel, SimulationError

from _util import graph_from_spec, make_graph, random_weighted_graph, spec_of


def _structure(spec):
    """A spec without its weights (ids, kinds, sizes, edges, byte counts)."""
    return {"root": spec["root"], "nodes": [r[:3] for r in spec["nodes"]],
            "edges": [r[:3] for r in spec["edges"]]}


def test_generator_reproduces_reference_graphs(small_cases, medium_cases):
    """generate_random_dag == the reference's (graph.py:180-305), structure only
    (the weights come from the device, tests/test_gpu_api_edges.py)."""
    for s in range(40):
        g = gen.generate_random_dag(*_small_shape(s), "MA", 256, seed=s)
        assert _structure(spec_of(g)) == _structure(small_cases[s]["spec"])
    for s, (n, m, kind) in enumerate([(38, 75, "MA"), (120, 240, "MA"), (120, 240, "MM"),
                                      (250, 500, "MA")]):
        gg = gen.generate_random_dag(n, m, kind, 1024, seed=s)
        assert _structure(spec_of(gg)) == _structure(medium_cases[s]["spec"])


def _small_shape(seed, max_kernels=15):
    """(n, m) of _util.random_weighted_graph(seed) (the reference's conftest recipe)."""
    import random
    from paper_1502_07451_b200.graph import InfeasibleGraphError
    rng = random.Random(seed)
    n = rng.randint(2, max_kernels)
    m = rng.randint(0, 2 * (n - 1))
    while True:
        try:
            gen.generate_random_dag(n, m, "MA", 256, seed=seed)
            return n, m
        except InfeasibleGraphError:
            m -= 1


def test_count_root_mode_matches_shape():
    g = gen.generate_random_dag(38, 75, "MA", 64, seed=3, count_root=True)
    assert len(g.nodes) == 38 and len(g.edges) == 75


def test_cholesky_dag_shape():
    g = gen.cholesky_dag(8)
    assert g.n_kernels() == 120
    assert len([e for e in g.edges if e[0] != 0]) == 252
    tasks, deps = gen.cholesky_tasks(64)
    assert len(tasks) == 45760 and len(deps) == 131040


@pytest.mark.gpu  # attach_weights runs on the device
def test_cholesky_matches_golden(medium_cases):
    c = [c for c in medium_cases if c["name"] == "cholesky_T8"][0]
    model = costs.load_calibration(
        "kind,size,time_cpu_ms,time_gpu_ms\nPOTRF,512,6.0,0.9\nTRSM,512,11.0,0.45\n"
        "SYRK,512,11.5,0.42\nGEMM,512,22.0,0.6\n[transfer]\nlatency_ms,bandwidth_bytes_per_ms\n"
        "0.01,12000000.0\n")
    assert spec_of(gen.cholesky_dag(8, model=model)) == c["spec"]


@pytest.mark.gpu  # topological_order runs on the device (hs_topological_order)
def test_topological_order_matches_golden(small_cases):
    for c in small_cases:
        assert topological_order(graph_from_spec(c["spec"])) == c["topological_order"]


@pytest.mark.gpu  # validate's cycle check is the device topological_order
def test_validate_messages():
    """Error substrings the reference's tests match (pkg/tests/test_graph.py:23-42)."""
    root = KernelNode(0, "SOURCE", 0)
    k1 = KernelNode(1, "K", 8, 1.0, 1.0)
    k2 = KernelNode(2, "K", 8, 1.0, 1.0)
    assert any("no edge from root" in p for p in validate(TaskGraph([root, k1], [])))
    g = TaskGraph([root, k1], [DataEdge(0, 1), DataEdge(1, 1)])
    assert any("self-loop" in p for p in validate(g))
    g = TaskGraph([root, k1, k2], [DataEdge(0, 1), DataEdge(1, 2), DataEdge(2, 1)])
    assert any("cycle" in p for p in validate(g))
    with pytest.raises(CycleError):
        topological_order(g)
    g = TaskGraph([root, KernelNode(1, "K", 8, -1.0, 1.0)], [DataEdge(0, 1)])
    assert any("negative" in p for p in validate(g))
    g = TaskGraph([KernelNode(0, "SOURCE", 0, 1.0, 0.0), k1], [DataEdge(0, 1)])
    assert any("zero weights" in p for p in validate(g))


def test_cost_model_known_answers():
    """pkg/tests/test_graph.py:123-141, test_costs.py:179-202."""
    m = costs.SyntheticCostModel()
    assert m.kernel_time("MA", 512, "CPU") == 0.81788928
    assert m.kernel_time("MA", 512, "GPU") == 0.2117152
    assert m.transfer_time(1024 * 1024 * 4) == 0.6965006451612903
    assert m.transfer_time(3 * 512 * 512 * 4) == 0.5273754838709678
    assert costs.speedup_ratio(m, "MM", 1024) == pytest.approx(40, rel=0.01)
    with pytest.raises(costs.UnknownKernelError):
        m.kernel_time("XX", 4, "CPU")
    with pytest.raises(costs.CostModelError):
        costs.PartitionTargets(0.3, 0.6)
    text = costs.dump_calibration(m)
    again = costs.load_calibration(text)
    assert again.kernel_time("MM", 1024, "GPU") == m.kernel_time("MM", 1024, "GPU")
    assert costs.dump_calibration(again) == text


def test_config_validation():
    with pytest.raises(PartitionError):
        PartitionConfig(node_weight_source="TPU")
    with pytest.raises(PartitionError):
        PartitionConfig(imbalance_tolerance=1.0)
    with pytest.raises(PartitionError):
        PartitionConfig(restarts=0)
    with pytest.raises(SimulationError):
        MachineModel(0, 0)
    with pytest.raises(SimulationError):
        MachineModel(-1, 1)


def test_unknown_policy_message():
    from paper_1502_07451_b200.policies import build_policy
    with pytest.raises(ValueError, match="unknown policy"):
        build_policy("fifo", make_graph({1: (1.0, 1.0)}, []))


def test_unit_weight_ugraph_host_side():
    """adjwgt=None (uniform edge weights, hs_ugraph_t.adjwgt_i = NULL): the
    materialised weights and the cut scale the partitioner's result uses."""
    import torch
    from paper_1502_07451_b200.kway import UGraph
    xadj = torch.tensor([0, 2, 3, 4], dtype=torch.int64)
    adj = torch.tensor([1, 2, 0, 0], dtype=torch.int32)
    vw = torch.ones(3, dtype=torch.int32)
    ug = UGraph(xadj, adj, None, vw, unit_weight=37)
    assert ug.weight_scale == 37 and ug.adjwgt.tolist() == [37] * 4
    ugw = UGraph(xadj, adj, torch.full((4,), 37, dtype=torch.int32), vw)
    assert ugw.weight_scale == 1 and torch.equal(ugw.adjwgt, ug.adjwgt)
