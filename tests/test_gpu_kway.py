"""Config 2/4 path on the device: generator, symmetrize, k-way partition, k-way evaluate,
levels — checked against the CPU oracle restatements."""
import numpy as np
import pytest
import torch

from paper_1502_07451_b200 import kway
from oracle import hetsched_oracle as O
from oracle import layered_oracle as LO

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,m,seed", [(50, 300, 0), (400, 4000, 3), (2000, 20000, 7)])
def test_generator_matches_oracle(n, m, seed):
    csr = kway.layered_dag(n, m, seed)
    preds, edges, layer = LO.generate(n, m, seed)
    src = np.repeat(np.arange(csr.n), np.diff(csr.out_ptr.cpu().numpy()))
    dst = csr.out_dst.cpu().numpy()
    assert list(zip(src.tolist(), dst.tolist())) == edges
    in_ptr = csr.in_ptr.cpu().numpy()
    in_src = csr.in_src.cpu().numpy()
    for v in range(csr.n):
        assert in_src[in_ptr[v]:in_ptr[v + 1]].tolist() == preds[v]
    in_eid = csr.in_eid.cpu().numpy()
    assert (dst[in_eid] == np.repeat(np.arange(csr.n), np.diff(in_ptr))).all()
    assert (src[in_eid] == in_src).all()
    lay = csr.layer_of.cpu().numpy()
    assert all(lay[v] == layer[v] for v in range(1, n + 1))


def test_dag_transpose_empty():
    from paper_1502_07451_b200.csr import DagCSR
    dev = torch.device("cuda")
    t = DagCSR.from_out_csr(0, torch.zeros(2, dtype=torch.int64, device=dev),
                            torch.zeros(0, dtype=torch.int32, device=dev))
    assert t.in_ptr.tolist() == [0, 0] and t.in_src.numel() == 0


@pytest.mark.parametrize("n,m,seed", [(2, 1, 0), (50, 300, 0), (3000, 30000, 5),
                                      (100000, 1000000, 9)])
def test_dag_transpose_matches_generator(n, m, seed):
    """hs_dag_transpose rebuilds the in-CSR (ascending sources, out-order ids) exactly."""
    from paper_1502_07451_b200.csr import DagCSR
    csr = kway.layered_dag(n, m, seed)
    t = DagCSR.from_out_csr(csr.root, csr.out_ptr, csr.out_dst)
    assert torch.equal(t.in_ptr, csr.in_ptr)
    assert torch.equal(t.in_src, csr.in_src)
    assert torch.equal(t.in_eid, csr.in_eid)


def _middle_root_dag(seed, n=400, m=3000):
    """HostDag whose root sits in the middle of the index order (kernel edges u < v)."""
    from paper_1502_07451_b200.csr import HostDag
    rng = np.random.default_rng(seed)
    root = n // 2
    kern = np.array([v for v in range(n) if v != root])
    pairs = set()
    while len(pairs) < m:
        a, b = sorted(rng.choice(kern, 2, replace=False).tolist())
        pairs.add((a, b))
    has_in = {b for _, b in pairs}
    pairs |= {(root, v) for v in kern.tolist() if v not in has_in}
    e = np.array(sorted(pairs), dtype=np.int32)
    ids = np.arange(n, dtype=np.int64)
    return HostDag(ids, root, e[:, 0].copy(), e[:, 1].copy(), rng.random(n), rng.random(n),
                   rng.random(len(e)), np.full(len(e), 4096, dtype=np.int64))


def test_dag_transpose_long_segments():
    """Fan-ins past the short (32) and CTA (4096) segment-sort limits."""
    from paper_1502_07451_b200.csr import DagCSR, HostDag
    n = 7000
    edges = {(0, v) for v in range(1, 5001)}
    edges |= {(u, 6001) for u in range(1, 5001)} | {(u, 6002) for u in range(4000, 4100)}
    edges |= {(u, 6003) for u in range(1, 40)} | {(6001, 6500), (6002, 6500)}
    edges |= {(0, v) for v in range(5001, n) if v not in (6001, 6002, 6003, 6500)}
    e = np.array(sorted(edges), dtype=np.int32)
    h = HostDag(np.arange(n, dtype=np.int64), 0, e[:, 0].copy(), e[:, 1].copy(), np.ones(n),
                np.ones(n), np.ones(len(e)), np.full(len(e), 8, dtype=np.int64))
    csr = DagCSR.from_host(h)
    t = DagCSR.from_out_csr(csr.root, csr.out_ptr, csr.out_dst)
    assert torch.equal(t.in_ptr, csr.in_ptr)
    assert torch.equal(t.in_src, csr.in_src)
    assert torch.equal(t.in_eid, csr.in_eid)


def test_dag_transpose_object_model_and_middle_root():
    """Object-model DAGs and a root in the middle of the id order, against the
    host lowering; K1 on the device-built CSC equals K1 on the host-built one."""
    from _util import random_weighted_graph
    from paper_1502_07451_b200.csr import DagCSR
    csrs = [DagCSR.from_taskgraph(random_weighted_graph(s, max_kernels=40)) for s in range(8)]
    csrs += [DagCSR.from_host(_middle_root_dag(s)) for s in range(3)]
    for csr in csrs:
        t = DagCSR.from_out_csr(csr.root, csr.out_ptr, csr.out_dst)
        assert torch.equal(t.in_ptr, csr.in_ptr)
        assert torch.equal(t.in_src, csr.in_src)
        assert torch.equal(t.in_eid, csr.in_eid)
        ew = kway.integer_weights(csr.w_xfer)
        nw = kway.integer_weights(csr.w_gpu)
        a, b = kway.symmetrize(csr, ew, nw), kway.symmetrize(t, ew, nw)
        assert torch.equal(a.xadj, b.xadj) and torch.equal(a.adjncy, b.adjncy)
        assert torch.equal(a.adjwgt, b.adjwgt) and torch.equal(a.vwgt, b.vwgt)
        xadj_e, adj_e, wgt_e = _expected_rows(csr, ew.cpu().numpy())
        assert (a.adjncy.cpu().numpy() == adj_e).all() and (a.adjwgt.cpu().numpy() == wgt_e).all()


def _host_graph(csr):
    src = np.repeat(np.arange(csr.n), np.diff(csr.out_ptr.cpu().numpy()))
    return src, csr.out_dst.cpu().numpy(), csr.bytes.cpu().numpy()


def test_symmetrize_adjacency_sets():
    csr = kway.layered_dag(3000, 30000, 1)
    ug = kway.symmetrize(csr)
    src, dst, _ = _host_graph(csr)
    keep = (src != 0) & (dst != 0)
    want = {}
    for u, v in zip(src[keep] - 1, dst[keep] - 1):
        want.setdefault(u, []).append(v)
        want.setdefault(v, []).append(u)
    xadj = ug.xadj.cpu().numpy()
    adj = ug.adjncy.cpu().numpy()
    assert ug.nnz == 2 * keep.sum()
    for v in range(ug.n):
        assert sorted(adj[xadj[v]:xadj[v + 1]].tolist()) == sorted(want.get(v, []))


def _expected_rows(csr, ew):
    """K1's exact entry sequence: per kernel, in-list (root dropped) then out-list."""
    op, od = csr.out_ptr.cpu().numpy(), csr.out_dst.cpu().numpy()
    ip, isrc = csr.in_ptr.cpu().numpy(), csr.in_src.cpu().numpy()
    ieid = csr.in_eid.cpu().numpy()
    root = csr.root
    adj, wgt, xadj = [], [], [0]
    for v in range(csr.n):
        if v == root:
            continue
        ins = [(u, ew[e]) for u, e in zip(isrc[ip[v]:ip[v + 1]], ieid[ip[v]:ip[v + 1]])
               if u != root]
        outs = list(zip(od[op[v]:op[v + 1]], ew[op[v]:op[v + 1]]))
        for u, w in ins + outs:
            adj.append(u if u < root else u - 1)
            wgt.append(w)
        xadj.append(len(adj))
    return np.array(xadj), np.array(adj), np.array(wgt)


@pytest.mark.parametrize("n,m", [(50, 300), (3000, 30000), (20011, 150007)])
def test_symmetrize_exact_sequence(n, m):
    """Chunked K1 writes the same entries in the same order as the per-vertex
    definition, with non-uniform weights (in-order copy or in_eid gather)."""
    csr = kway.layered_dag(n, m, 2)
    ew = torch.randint(1, 1000, (csr.m,), dtype=torch.int32, device=csr.device)
    xadj_e, adj_e, wgt_e = _expected_rows(csr, ew.cpu().numpy())
    for w_in in (None, kway.in_order(csr, ew)):
        ug = kway.symmetrize(csr, ew, None, w_in)
        assert ug.weight_scale == 1
        assert (ug.xadj.cpu().numpy() == xadj_e).all()
        assert (ug.adjncy.cpu().numpy() == adj_e).all()
        assert (ug.adjwgt.cpu().numpy() == wgt_e).all()


def test_uniform_weights_unit_path_identical(monkeypatch):
    """Uniform edge weights: K1 writes no weight stream (adjwgt NULL = unit
    weights) and the partition and cut equal the explicit-weight run's."""
    csr = kway.layered_dag(20000, 200000, 4)
    ew = torch.full((csr.m,), 37, dtype=torch.int32, device=csr.device)
    ug = kway.symmetrize(csr, ew)
    assert ug._adjwgt is None and ug.weight_scale == 37
    monkeypatch.setenv("HS_KWAY_WEIGHTS", "1")
    ugw = kway.symmetrize(csr, ew)
    assert ugw._adjwgt is not None
    assert (ugw.adjncy == ug.adjncy).all() and (ugw.adjwgt == ug.adjwgt).all()
    r = kway.partition_kway(ug, 8, tol=0.03, seed=3)
    rw = kway.partition_kway(ugw, 8, tol=0.03, seed=3)
    assert (r.part == rw.part).all() and r.cut == rw.cut
    p = r.part.long()
    src = torch.repeat_interleave(torch.arange(ug.n, device=p.device), ug.xadj.diff())
    assert r.cut == int(((p[src] != p[ug.adjncy.long()]).sum().item() // 2) * 37)


@pytest.mark.parametrize("n,m,k", [(5000, 50000, 2), (20000, 200000, 8), (100000, 1000000, 8),
                                   (100000, 1000000, 3), (100000, 1000000, 16),
                                   (200000, 2000000, 32)])
def test_kway_valid_balanced_deterministic(n, m, k):
    csr = kway.layered_dag(n, m, 0)
    ug = kway.symmetrize(csr)
    r1 = kway.partition_kway(ug, k, tol=0.03, seed=5)
    r2 = kway.partition_kway(ug, k, tol=0.03, seed=5)
    p1 = r1.part.cpu().numpy()
    assert (p1 == r2.part.cpu().numpy()).all(), "not deterministic"
    assert p1.min() >= 0 and p1.max() < k
    assert r1.feasible and r1.max_deviation <= 0.03
    # the reported deviation is the one of the returned parts (the finest
    # refinement's running part weights stand in for a final recount)
    vw = ug.vwgt.cpu().numpy().astype(np.int64)
    pw = np.bincount(p1, weights=vw, minlength=k)
    dev = float(np.abs(pw / float(vw.sum()) - 1.0 / k).max())
    assert abs(r1.max_deviation - dev) <= 2e-9
    # integer cut from the partitioner == K2 on the directed DAG == oracle
    nodep = kway.kernel_to_node_parts(csr, r1.part)
    ev = kway.evaluate_batch(csr, nodep.unsqueeze(0), k,
                             node_w_i=kway.integer_weights(csr.w_gpu).to(torch.int64))
    src, dst, nb = _host_graph(csr)
    ew = kway.integer_weights(csr.w_xfer).cpu().numpy()
    np_ = nodep.cpu().numpy()
    cut_w = int(ew[(src != 0) & (dst != 0) & (np_[src] != np_[dst])].sum())
    assert r1.cut == cut_w
    vw = kway.integer_weights(csr.w_gpu).cpu().numpy()
    ref = O.evaluate_kway(csr.n, 0, src.tolist(), dst.tolist(), nb.tolist(), np_.tolist(), k, vw)
    for key in ("cut_bytes", "cut_edges", "xfer_count", "xfer_bytes"):
        assert int(ev[key][0]) == ref[key], key
    assert ev["loads"][0].cpu().tolist() == ref["loads"]
    # quality: clearly better than a random balanced assignment
    rnd = np.random.default_rng(0).integers(0, k, size=ug.n)
    nodes_r = np.concatenate([[0], rnd])
    rand_cut = int(ew[(src != 0) & (dst != 0) & (nodes_r[src] != nodes_r[dst])].sum())
    assert r1.cut < rand_cut


def test_levels_and_critical_path_match_oracle():
    csr = kway.layered_dag(3000, 20000, 2)
    lv, finish, cp, nl = kway.levels(csr)
    src, dst, _ = _host_graph(csr)
    nodes = [[i, "MA", 512, float(csr.w_cpu[i]), float(csr.w_gpu[i])] for i in range(csr.n)]
    wx = csr.w_xfer.cpu().numpy()
    spec = {"root": 0, "nodes": nodes,
            "edges": [[int(u), int(v), 0, float(w)] for u, v, w in zip(src, dst, wx)]}
    g = O.OGraph(spec)
    assert cp == O.critical_path(g)
    want = O.levels(g)
    got = lv.cpu().numpy()
    assert all(got[i] == want[i] for i in range(csr.n))
    order = kway.level_order(csr).cpu().numpy().tolist()
    assert order == O.level_order(g)


def test_assigned_makespan_matches_oracle(small_cases):
    """K7 mode 3 (level-synchronous makespan of a given assignment) vs the oracle, bit-exact."""
    import random
    from oracle import hetsched_oracle as O
    from paper_1502_07451_b200.csr import DagCSR
    from _util import graph_from_spec
    rng = random.Random(5)
    for case in small_cases[:25]:
        g = graph_from_spec(case["spec"])
        og = O.OGraph(case["spec"])
        csr = DagCSR.from_taskgraph(g)
        ids = [int(i) for i in csr.ids]
        for k, gpu_parts in ((2, {1}), (4, {1, 2, 3}), (3, {0})):
            part = {nid: rng.randrange(k) for nid in ids}
            dev_part = torch.tensor([part[i] for i in ids], dtype=torch.int32, device="cuda")
            ms, _ = kway.assigned_makespan(csr, dev_part, sorted(gpu_parts), k=k)
            assert ms == O.assigned_makespan(og, part, gpu_parts)


def test_assigned_makespan_layered_partition():
    """20k/200k layered DAG partitioned k=8: device makespan == oracle restatement."""
    from oracle import hetsched_oracle as O
    csr = kway.layered_dag(20_000, 200_000, seed=9)
    r = kway.partition_kway(csr, 8, seed=0)
    node_part = kway.kernel_to_node_parts(csr, r.part)
    ms, fin = kway.assigned_makespan(csr, node_part, k=8)
    out_ptr = csr.out_ptr.cpu().numpy()
    dst = csr.out_dst.cpu().numpy()
    wx = csr.w_xfer.cpu().numpy()
    wc, wg = csr.w_cpu.cpu().numpy(), csr.w_gpu.cpu().numpy()
    spec = {"root": 0, "nodes": [[i, "MA", 512, float(wc[i]), float(wg[i])] for i in range(csr.n)],
            "edges": [[u, int(dst[e]), 0, float(wx[e])] for u in range(csr.n)
                      for e in range(out_ptr[u], out_ptr[u + 1])]}
    spec["nodes"][0][1] = "SOURCE"
    p = node_part.cpu().numpy()
    want = O.assigned_makespan(O.OGraph(spec), {i: int(p[i]) for i in range(csr.n)},
                               set(range(8)))
    assert ms == want and ms > 0


@pytest.mark.parametrize("n,m", [(3000, 20000), (200_000, 2_000_000)])
def test_levels_dataflow_equals_frontier(n, m):
    """K7 on a creation-order DAG (every edge points up: the barrier-free
    dataflow kernel) equals K7 on the same DAG randomly renumbered (the
    frontier kernel), node for node under the permutation: levels, finish
    times (bits), critical path; and mode 3 on an assignment."""
    csr = kway.layered_dag(n, m, seed=4)
    rel, pi = kway.relabeled_dag(csr, seed=2)
    lv, fin, cp, nl = kway.levels(csr)
    lv2, fin2, cp2, nl2 = kway.levels(rel)
    pil = pi.long()
    assert cp == cp2 and nl == nl2
    assert torch.equal(lv2[pil], lv) and torch.equal(fin2[pil], fin)
    part = torch.randint(0, 4, (csr.n,), dtype=torch.int32, device=csr.device)
    part2 = torch.empty_like(part)
    part2[pil] = part
    ms, f1 = kway.assigned_makespan(csr, part, [1, 3], k=4)
    ms2, f2 = kway.assigned_makespan(rel, part2, [1, 3], k=4)
    assert ms == ms2 and torch.equal(f2[pil], f1)


def test_connectivity_cache_is_exact():
    """The finest-level connectivity cache (kept exact by every applied move,
    L2-hinted) gives the same partition as rescanning the adjacency every
    pass (HS_KWAY_NOCACHE=1): config-2 shape, uniform and U[1,100] weights."""
    import os
    csr = kway.layered_dag(100_000, 1_000_000, seed=6)
    g = torch.Generator(device="cpu").manual_seed(3)
    ew = torch.randint(1, 101, (csr.m,), generator=g, dtype=torch.int32).to(csr.device)
    nw = torch.randint(1, 101, (csr.n,), generator=g, dtype=torch.int32).to(csr.device)
    for ug in (kway.symmetrize(csr), kway.symmetrize(csr, ew, nw)):
        a = kway.partition_kway(ug, 8, seed=1)
        os.environ["HS_KWAY_NOCACHE"] = "1"
        try:
            b = kway.partition_kway(ug, 8, seed=1)
        finally:
            del os.environ["HS_KWAY_NOCACHE"]
        assert a.cut == b.cut and torch.equal(a.part, b.part)
