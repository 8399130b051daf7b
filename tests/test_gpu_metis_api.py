"""METIS_PartGraphKway-compatible C entry point, called through ctypes like a METIS user."""
import ctypes

import numpy as np
import pytest

from paper_1502_07451_b200 import _native

pytestmark = pytest.mark.gpu


def test_metis_signature_partitions_a_grid():
    # 2D 40x40 grid graph in METIS CSR (0-based), unit weights
    w = 40
    n = w * w
    xadj, adj = [0], []
    for r in range(w):
        for c in range(w):
            for dr, dc in ((-1, 0), (1, 0), (0, -1), (0, 1)):
                rr, cc = r + dr, c + dc
                if 0 <= rr < w and 0 <= cc < w:
                    adj.append(rr * w + cc)
            xadj.append(len(adj))
    I = ctypes.c_int32
    arr = lambda a: (I * len(a))(*a)  # noqa: E731
    nv, ncon, nparts = I(n), I(1), I(4)
    part = (I * n)()
    obj = I(0)
    fn = _native._lib.hs_METIS_PartGraphKway
    fn.restype = ctypes.c_int
    rc = fn(ctypes.byref(nv), ctypes.byref(ncon), arr(xadj), arr(adj), None, None, None,
            ctypes.byref(nparts), None, None, None, ctypes.byref(obj), part)
    assert rc == 0, _native._lib.hs_last_error()
    p = np.array(part[:])
    assert p.min() >= 0 and p.max() < 4
    sizes = np.bincount(p, minlength=4)
    assert abs(sizes / n - 0.25).max() <= 0.25 * 0.03 + 1e-9
    cut = sum(1 for v in range(n) for j in range(xadj[v], xadj[v + 1]) if p[v] != p[adj[j]]) // 2
    assert obj.value == cut
    assert cut < 0.5 * len(adj) // 2  # far better than random (~75% of edges)
