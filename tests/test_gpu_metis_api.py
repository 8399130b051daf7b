"""METIS_PartGraphKway-compatible C entry point, called through ctypes like a METIS user."""
import ctypes

import numpy as np
import pytest

from paper_1502_07451_b200 import _native

pytestmark = pytest.mark.gpu

I = ctypes.c_int32
METIS_OK, METIS_ERROR_INPUT = 1, -2


def grid_graph(w):
    xadj, adj = [0], []
    for r in range(w):
        for c in range(w):
            for dr, dc in ((-1, 0), (1, 0), (0, -1), (0, 1)):
                rr, cc = r + dr, c + dc
                if 0 <= rr < w and 0 <= cc < w:
                    adj.append(rr * w + cc)
            xadj.append(len(adj))
    return xadj, adj


def arr(a):
    return (I * len(a))(*a)


def call(fn_name, n, xadj, adj, nparts, options=None, adjwgt=None):
    fn = getattr(_native._lib, fn_name)
    fn.restype = ctypes.c_int
    nv, ncon, npt = I(n), I(1), I(nparts)
    part = (I * n)()
    obj = I(0)
    rc = fn(ctypes.byref(nv), ctypes.byref(ncon), arr(xadj), arr(adj), None, None,
            arr(adjwgt) if adjwgt is not None else None, ctypes.byref(npt), None, None,
            arr(options) if options is not None else None, ctypes.byref(obj), part)
    return rc, np.array(part[:]), obj.value


@pytest.mark.parametrize("fn_name", ["METIS_PartGraphKway", "hs_METIS_PartGraphKway"])
def test_metis_signature_partitions_a_grid(fn_name):
    # 2D 40x40 grid graph in METIS CSR (0-based), unit weights
    w = 40
    n = w * w
    xadj, adj = grid_graph(w)
    rc, p, obj = call(fn_name, n, xadj, adj, 4)
    assert rc == METIS_OK, _native._lib.hs_last_error()
    assert p.min() >= 0 and p.max() < 4
    sizes = np.bincount(p, minlength=4)
    assert abs(sizes / n - 0.25).max() <= 0.25 * 0.03 + 1e-9
    cut = sum(1 for v in range(n) for j in range(xadj[v], xadj[v + 1]) if p[v] != p[adj[j]]) // 2
    assert obj == cut
    assert cut < 0.5 * len(adj) // 2  # far better than random (~75% of edges)


def test_metis_fortran_numbering_and_seed_option():
    w = 24
    n = w * w
    xadj, adj = grid_graph(w)
    opts = [-1] * 40
    opts[17] = 1  # METIS_OPTION_NUMBERING: 1-based
    opts[8] = 5   # METIS_OPTION_SEED
    rc1, p1, obj1 = call("METIS_PartGraphKway", n, [x + 1 for x in xadj], [a + 1 for a in adj], 3,
                         options=opts)
    assert rc1 == METIS_OK
    assert p1.min() == 1 and p1.max() == 3
    opts[17] = 0
    rc0, p0, obj0 = call("METIS_PartGraphKway", n, xadj, adj, 3, options=opts)
    assert rc0 == METIS_OK
    assert np.array_equal(p1 - 1, p0) and obj0 == obj1


def test_metis_weighted_edges_objval():
    w = 20
    n = w * w
    xadj, adj = grid_graph(w)
    # edge weight = 1 + (min(u, v) % 3), symmetric
    wts = []
    for v in range(n):
        for j in range(xadj[v], xadj[v + 1]):
            wts.append(1 + min(v, adj[j]) % 3)
    rc, p, obj = call("METIS_PartGraphKway", n, xadj, adj, 2, adjwgt=wts)
    assert rc == METIS_OK
    cut = sum(wts[j] for v in range(n) for j in range(xadj[v], xadj[v + 1])
              if p[v] != p[adj[j]]) // 2
    assert obj == cut


def test_metis_bad_input_returns_error_input():
    xadj, adj = grid_graph(4)
    bad = list(adj)
    bad[3] = 99  # neighbour out of range
    rc, _, _ = call("METIS_PartGraphKway", 16, xadj, bad, 2)
    assert rc == METIS_ERROR_INPUT
    assert b"out of range" in _native._lib.hs_last_error()
