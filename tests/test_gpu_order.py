"""Band-start vertex orders (csrc/order.cu): topological check, level permutation,
relabelled kernel graph, and the id-order robustness of ``partition_dag``."""
import numpy as np
import pytest
import torch

from paper_1502_07451_b200 import _native, kway

pytestmark = pytest.mark.gpu


def _int_cut(csr, kpart_node, ew):
    """Integer cut of a node-space part array over the DAG's kernel edges."""
    src = torch.repeat_interleave(torch.arange(csr.n, device=csr.device), csr.out_ptr.diff())
    dst = csr.out_dst.long()
    keep = (src != csr.root) & (dst != csr.root)
    diff = kpart_node[src] != kpart_node[dst]
    return int(ew[keep & diff].long().sum().item())


def test_topological_flag():
    csr = kway.layered_dag(5000, 50000, 2)
    assert _native.dag_is_topological(csr)
    rel, _ = kway.relabeled_dag(csr, seed=3)
    assert not _native.dag_is_topological(rel)


def test_level_permutation_is_stable_level_sort():
    csr = kway.layered_dag(20000, 200000, 1)
    rel, _ = kway.relabeled_dag(csr, seed=4)
    lv, _, _, nl = _native.levels(rel, 0)
    perm, inv = _native.level_permutation(rel, lv, nl)
    lvn = lv.cpu().numpy()
    root = rel.root
    klev = np.delete(lvn, root)
    expect = np.argsort(klev, kind="stable")
    assert (perm.cpu().numpy() == expect).all()
    assert (inv.cpu().numpy()[expect] == np.arange(len(expect))).all()


def test_ugraph_permute_matches_numpy():
    csr = kway.layered_dag(3000, 30000, 5)
    ew = kway.integer_weights(csr.w_xfer)
    ew[::7] += 3  # non-uniform weights: the weight stream is permuted too
    ug = kway.symmetrize(csr, ew)
    g = torch.Generator().manual_seed(0)
    perm = torch.randperm(ug.n, generator=g).to(torch.int32).cuda()
    inv = torch.empty_like(perm)
    inv[perm.long()] = torch.arange(ug.n, dtype=torch.int32, device=perm.device)
    pg = kway.permute_ugraph(ug, perm, inv)
    x, a, w, vw = (t.cpu().numpy() for t in (ug.xadj, ug.adjncy, ug.adjwgt, ug.vwgt))
    px, pa, pw, pvw = (t.cpu().numpy() for t in (pg.xadj, pg.adjncy, pg.adjwgt, pg.vwgt))
    p, iv = perm.cpu().numpy(), inv.cpu().numpy()
    assert (pvw == vw[p]).all()
    for i in range(0, ug.n, 37):
        o = p[i]
        got = sorted(zip(pa[px[i]:px[i + 1]].tolist(), pw[px[i]:px[i + 1]].tolist()))
        exp = sorted(zip(iv[a[x[o]:x[o + 1]]].tolist(), w[x[o]:x[o + 1]].tolist()))
        assert got == exp


@pytest.mark.parametrize("n,m", [(100_000, 1_000_000), (20_000, 200_000)])
def test_relabelled_dag_partition(n, m):
    """A random numbering of the same DAG: feasible, cut within 1% of (or below)
    the generated numbering's, parts indexed by the relabelled kernel positions."""
    csr = kway.layered_dag(n, m, 0)
    r0 = kway.partition_dag(csr, 8, tol=0.03)
    rel, pi = kway.relabeled_dag(csr, seed=1)
    r1 = kway.partition_dag(rel, 8, tol=0.03)
    r2 = kway.partition_dag(rel, 8, tol=0.03)
    assert torch.equal(r1.part, r2.part), "not deterministic"
    assert r1.feasible and r1.max_deviation <= 0.03
    assert r1.cut <= 1.01 * r0.cut, (r1.cut, r0.cut)
    ew = kway.integer_weights(rel.w_xfer)
    node = kway.kernel_to_node_parts(rel, r1.part)
    assert _int_cut(rel, node, ew) == r1.cut
    p = r1.part.cpu().numpy()
    assert p.min() >= 0 and p.max() < 8


def test_partition_dag_order_ids_equals_partition_kway():
    csr = kway.layered_dag(20000, 200000, 3)
    a = kway.partition_dag(csr, 4, tol=0.03, order="ids", seed=2)
    b = kway.partition_kway(kway.symmetrize(csr), 4, tol=0.03, seed=2)
    assert torch.equal(a.part, b.part) and a.cut == b.cut
