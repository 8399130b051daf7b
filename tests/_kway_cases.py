"""Integer-weighted graphs of the k-way quality tests (test infrastructure).

Each case is (n, eu, ev, ew, vw): n vertices (kernel positions), undirected
edges eu < ev with integer weight ew, integer vertex weights vw — the graph
``kway.symmetrize`` derives from a task DAG with the METIS integerisation
``_scaled(w, 100)`` (graphio.py:272-274). Built on the CPU only, so the golden
script (which runs the REFERENCE partitioner on the same arrays,
tests/golden/make_kway_golden.py) and the GPU tests see identical inputs; the
fixture stores a sha256 of the arrays and the tests check it.
"""
from __future__ import annotations

import hashlib
import json
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from oracle import layered_oracle  # noqa: E402

# the reference's synthetic cost model for MA-512 (costs.py:82-143; known
# answers pkg/tests/test_graph.py:123-141) and the calibration of the
# tiled-Cholesky DAG used by tests/golden/make_golden.py
CHOL = {"POTRF": 0.9, "TRSM": 0.45, "SYRK": 0.42, "GEMM": 0.6}
CHOL_XFER = 0.01 + (512 * 512 * 8) / 12_000_000.0


def scaled(w: float, scale: int = 100) -> int:
    """graphio.py:272-274"""
    return max(1, int(math.floor(w * scale + 0.5)))


def _ma512():
    from paper_1502_07451_b200.costs import SyntheticCostModel
    m = SyntheticCostModel()
    return m.kernel_time("MA", 512, "GPU"), m.transfer_time(512 * 512 * 4)


def layered(n, m, seed, uniform_rng=None):
    preds, edges, _ = layered_oracle.generate(n, m, seed)
    inter = [(u - 1, v - 1) for (u, v) in edges if u != 0]
    eu = np.array([a for a, _ in inter], dtype=np.int64)
    ev = np.array([b for _, b in inter], dtype=np.int64)
    if uniform_rng is None:
        wg, wx = _ma512()
        vw = np.full(n, scaled(wg), dtype=np.int64)
        ew = np.full(len(eu), scaled(wx), dtype=np.int64)
    else:
        rng = np.random.default_rng(uniform_rng)
        vw = rng.integers(1, 101, size=n).astype(np.int64)
        ew = rng.integers(1, 101, size=len(eu)).astype(np.int64)
    return n, eu, ev, ew, vw


def cholesky(tiles):
    from paper_1502_07451_b200.gen import cholesky_tasks
    tasks, deps = cholesky_tasks(tiles)
    n = len(tasks)
    vw = np.array([scaled(CHOL[kind]) for kind, _ in tasks], dtype=np.int64)
    eu = np.array([u - 1 for u, _ in deps], dtype=np.int64)
    ev = np.array([v - 1 for _, v in deps], dtype=np.int64)
    ew = np.full(len(deps), scaled(CHOL_XFER), dtype=np.int64)
    return n, eu, ev, ew, vw


def from_spec(spec):
    root = spec["root"]
    ids = sorted(int(r[0]) for r in spec["nodes"] if int(r[0]) != root)
    pos = {i: k for k, i in enumerate(ids)}
    wg = {int(r[0]): float(r[4]) for r in spec["nodes"]}
    vw = np.array([scaled(wg[i]) for i in ids], dtype=np.int64)
    es = [(pos[int(u)], pos[int(v)], scaled(float(w))) for u, v, _, w in spec["edges"]
          if int(u) != root and int(v) != root]
    eu = np.array([a for a, _, _ in es], dtype=np.int64)
    ev = np.array([b for _, b, _ in es], dtype=np.int64)
    ew = np.array([w for _, _, w in es], dtype=np.int64)
    return len(ids), eu, ev, ew, vw


def cases():
    out = {
        "L200": lambda: layered(200, 2000, 0),
        "L300": lambda: layered(300, 3000, 2),
        "L500": lambda: layered(500, 5000, 1),
        "L1000": lambda: layered(1000, 10000, 3),
        "L2000": lambda: layered(2000, 20000, 4),
        "LU500": lambda: layered(500, 5000, 5, uniform_rng=5),
        "LU1000": lambda: layered(1000, 10000, 6, uniform_rng=6),
        "CH16": lambda: cholesky(16),
    }
    with open(os.path.join(ROOT, "tests", "golden", "medium_graphs.json")) as f:
        for c in json.load(f):
            out[c["name"]] = (lambda spec: (lambda: from_spec(spec)))(c["spec"])
    return out


def digest(case) -> str:
    n, eu, ev, ew, vw = case
    h = hashlib.sha256()
    h.update(np.int64(n).tobytes())
    for a in (eu, ev, ew, vw):
        h.update(np.ascontiguousarray(a, dtype=np.int64).tobytes())
    return h.hexdigest()


def csr(case):
    """Symmetric CSR (xadj int64, adjncy int32, adjwgt int32, vwgt int32) of a case."""
    n, eu, ev, ew, vw = case
    src = np.concatenate([eu, ev])
    dst = np.concatenate([ev, eu])
    w = np.concatenate([ew, ew])
    o = np.lexsort((dst, src))
    src, dst, w = src[o], dst[o], w[o]
    xadj = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(src, minlength=n), out=xadj[1:])
    return xadj, dst.astype(np.int32), w.astype(np.int32), vw.astype(np.int32)


def int_cut(case, part) -> int:
    n, eu, ev, ew, vw = case
    part = np.asarray(part)
    return int(ew[part[eu] != part[ev]].sum())


def max_dev(case, part, k) -> float:
    """max_p |w_p / W - 1/k| in doubles (the k-way form of partition.py:72)."""
    vw = case[4]
    W = float(vw.sum())
    part = np.asarray(part)
    return max(abs(float(vw[part == p].sum()) / W - 1.0 / k) for p in range(k))
