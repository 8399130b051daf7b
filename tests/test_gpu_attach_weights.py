"""Device weight attachment (hs_attach_weights) against the REFERENCE.

attach_weights (graph.py:308-324) with the synthetic model (MA/MM closed
forms per node on the device) and a calibration table (values read once per
(kind, size)) reproduces the golden graphs the unmodified reference built
(tests/golden/small_graphs.json, medium_graphs.json: generate_random_dag +
attach_weights, and the tiled-Cholesky DAG with its calibration CSV) bit for
bit; the reference's known answers (pkg/tests/test_graph.py:123-141); its
error behaviour (GraphError with the model's message for the first node in
node order without a cost entry; CostModelError for a negative byte count);
custom duck-typed models; and the CSR path on config-2-sized graphs.
"""
import numpy as np
import pytest
import torch

from _util import random_weighted_graph, spec_of

pytestmark = pytest.mark.gpu


def test_generated_graphs_match_reference(small_cases, medium_cases):
    from paper_1502_07451_b200 import costs, gen
    from paper_1502_07451_b200.graph import attach_weights
    for s in range(40):
        assert spec_of(random_weighted_graph(s)) == small_cases[s]["spec"]
    for s in range(10):
        g = random_weighted_graph(100 + s, kind="MM", size=1024)
        assert spec_of(g) == small_cases[40 + s]["spec"]
    for s, (n, m, kind) in enumerate([(38, 75, "MA"), (120, 240, "MA"), (120, 240, "MM"),
                                      (250, 500, "MA")]):
        gg = gen.generate_random_dag(n, m, kind, 1024, seed=s)
        assert spec_of(attach_weights(gg, costs.SyntheticCostModel())) == medium_cases[s]["spec"]


def test_known_answers():
    """pkg/tests/test_graph.py:123-141"""
    from paper_1502_07451_b200.costs import SyntheticCostModel
    from paper_1502_07451_b200.graph import DataEdge, KernelNode, TaskGraph, attach_weights
    g = TaskGraph([KernelNode(0, "SOURCE", 0), KernelNode(1, "MA", 512), KernelNode(2, "MA", 1024)],
                  [DataEdge(0, 1), DataEdge(1, 2, bytes=4194304)])
    w = attach_weights(g, SyntheticCostModel())
    assert w.nodes[1].weight_cpu == 0.81788928 and w.nodes[1].weight_gpu == 0.2117152
    assert w.edges[(1, 2)].weight_xfer == 0.6965006451612903
    assert w.nodes[0].weight_cpu == 0.0 and w.edges[(0, 1)].weight_xfer == 0.02


def test_calibration_table_and_interpolation(medium_cases):
    from paper_1502_07451_b200 import costs, gen
    from paper_1502_07451_b200.graph import DataEdge, KernelNode, TaskGraph, attach_weights
    csv = ("kind,size,time_cpu_ms,time_gpu_ms\nPOTRF,512,6.0,0.9\nTRSM,512,11.0,0.45\n"
           "SYRK,512,11.5,0.42\nGEMM,512,22.0,0.6\n[transfer]\nlatency_ms,bandwidth_bytes_per_ms\n"
           "0.01,12000000.0\n")
    c = [c for c in medium_cases if c["name"] == "cholesky_T8"][0]
    assert spec_of(gen.cholesky_dag(8, model=costs.load_calibration(csv))) == c["spec"]
    interp = costs.load_calibration(
        "kind,size,time_cpu_ms,time_gpu_ms\nMM,256,1.0,0.5\nMM,1024,9.0,0.7\n[transfer]\n"
        "latency_ms,bandwidth_bytes_per_ms\n0.03,7000000.0\n", interpolate=True)
    g = TaskGraph([KernelNode(0, "SOURCE", 0)] + [KernelNode(i, "MM", s) for i, s in
                                                  enumerate([256, 300, 777, 1024], 1)],
                  [DataEdge(0, i, bytes=8 * i) for i in range(1, 5)])
    w = attach_weights(g, interp)
    for i in range(1, 5):
        n = g.nodes[i]
        assert w.nodes[i].weight_cpu == interp.kernel_time("MM", n.size, "CPU")
        assert w.nodes[i].weight_gpu == interp.kernel_time("MM", n.size, "GPU")
        assert w.edges[(0, i)].weight_xfer == interp.transfer_time(8 * i)


def test_errors_follow_reference():
    from paper_1502_07451_b200.costs import CostModelError, SyntheticCostModel
    from paper_1502_07451_b200.graph import (DataEdge, GraphError, KernelNode, TaskGraph,
                                             attach_weights)
    # node order, not id order: kernel 7 comes first
    g = TaskGraph([KernelNode(0, "SOURCE", 0), KernelNode(7, "FFT", 64), KernelNode(2, "XX", 8)],
                  [DataEdge(0, 7), DataEdge(0, 2)])
    with pytest.raises(GraphError, match=r"no cost entry for kernel 7 \(FFT, 64\): synthetic"):
        attach_weights(g, SyntheticCostModel())
    g = TaskGraph([KernelNode(0, "SOURCE", 0), KernelNode(1, "MA", 64)],
                  [DataEdge(0, 1), DataEdge(1, 1, bytes=-4)])
    with pytest.raises(CostModelError, match="negative byte count"):
        attach_weights(g, SyntheticCostModel())


def test_custom_model_and_large_sizes():
    from paper_1502_07451_b200.costs import SyntheticCostModel
    from paper_1502_07451_b200.graph import DataEdge, KernelNode, TaskGraph, attach_weights

    class Custom:
        def kernel_time(self, kind, size, device):
            return (size * 0.5 + (1.0 if device == "GPU" else 3.0)) / 7.0

        def transfer_time(self, nbytes):
            return nbytes / 3.0 + 0.1

    sizes = [1, 3, 1000, 2 ** 20, 2 ** 27 + 1, 2 ** 30 + 7]
    g = TaskGraph([KernelNode(0, "SOURCE", 0)] + [KernelNode(i, k, s) for i, s in enumerate(sizes, 1)
                                                  for k in ["MM"]],
                  [DataEdge(0, i, bytes=13 * i) for i in range(1, len(sizes) + 1)])
    for model in (Custom(), SyntheticCostModel()):
        w = attach_weights(g, model)
        for i, s in enumerate(sizes, 1):
            assert w.nodes[i].weight_cpu == model.kernel_time("MM", s, "CPU")
            assert w.nodes[i].weight_gpu == model.kernel_time("MM", s, "GPU")
            assert w.edges[(0, i)].weight_xfer == model.transfer_time(13 * i)


def test_csr_weights_config2():
    """The CSR path on a 100k/1M layered DAG with mixed kinds and sizes:
    every weight equals the model's own scalar answer."""
    from paper_1502_07451_b200 import costs, kway
    csr = kway.layered_dag(100_000, 1_000_000, seed=0)
    n, m = csr.n, csr.m
    gen_ = torch.Generator(device="cpu").manual_seed(1)
    kinds = ["MA", "MM"]
    kcode = torch.randint(0, 2, (n,), generator=gen_, dtype=torch.int32)
    sizes = torch.tensor([64, 256, 512, 1024], dtype=torch.int64)[
        torch.randint(0, 4, (n,), generator=gen_)]
    model = costs.SyntheticCostModel()
    kway.attach_weights_csr(csr, kcode.to(csr.device), kinds, sizes.to(csr.device), model)
    wc, wg, wx = (t.cpu().numpy() for t in (csr.w_cpu, csr.w_gpu, csr.w_xfer))
    kc, sz = kcode.numpy(), sizes.numpy()
    for v in np.random.default_rng(0).integers(0, n, 2000):
        if v == csr.root:
            assert wc[v] == 0.0 and wg[v] == 0.0
            continue
        assert wc[v] == model.kernel_time(kinds[kc[v]], int(sz[v]), "CPU")
        assert wg[v] == model.kernel_time(kinds[kc[v]], int(sz[v]), "GPU")
    b = csr.bytes.cpu().numpy()
    for e in np.random.default_rng(1).integers(0, m, 2000):
        assert wx[e] == model.transfer_time(int(b[e]))
