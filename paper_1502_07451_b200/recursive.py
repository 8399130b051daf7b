"""The reference heuristic as a k-way start: recursive bisection by ``partition_heuristic``.

The reference partitions 2-way only (partition.py:258-295; k > 2 is a
non-goal). Applied recursively — split the part range [p0, p1) at
pm = p0 + (p1 - p0) // 2 with r_cpu = t[p0:pm] / t[p0:p1], CPU side = the lower
half — it is the natural k-way baseline the k-way partitioner must match or
beat. This module computes that recursion on the device with
the exact 2-way kernel (csrc/fm2.cu, bit-exact with the reference: greedy
fill, balance repair, FM passes, 1 + restarts start orders, winner by
(not feasible, cut, err, lex)), one batched launch per recursion depth.

``kway.partition_kway`` hands the result to the k-way partitioner as a start
partition (``hs_partition_kway_starts``) for graphs of at most
``MAX_KERNELS`` vertices; the partitioner FM-refines it next to its own
candidates and keeps the best, so its cut is never above this baseline's at
the same balance constraint.

Weights are the graph's integer weights (as fp64), so every sum the 2-way
kernel forms is exact and the adjacency order of a subgraph cannot change a
decision; vertex positions ascend like the reference's sorted kernel ids.
"""
from __future__ import annotations

from typing import List, Optional, Sequence, Tuple

import numpy as np
import torch

from . import _native
from .csr import HostDag, TwoWayBatch
from .partition import PartitionConfig, start_orders

MAX_KERNELS = 2048


def _undirected_edges(xadj: np.ndarray, adjncy: np.ndarray, adjwgt: np.ndarray):
    """Each undirected edge once as (u < v, w), sorted by (u, v)."""
    n = len(xadj) - 1
    src = np.repeat(np.arange(n, dtype=np.int64), np.diff(xadj))
    keep = adjncy > src
    u, v, w = src[keep], adjncy[keep].astype(np.int64), adjwgt[keep].astype(np.float64)
    o = np.lexsort((v, u))
    return u[o], v[o], w[o]


def _subgraph(members: np.ndarray, eu, ev, ew, vw: np.ndarray) -> HostDag:
    """HostDag of the induced subgraph: root 0, kernels 1..len(members) in member order."""
    pos = np.full(len(vw), -1, dtype=np.int64)
    pos[members] = np.arange(1, len(members) + 1)
    keep = (pos[eu] > 0) & (pos[ev] > 0)
    su, sv, sw = pos[eu[keep]], pos[ev[keep]], ew[keep]
    o = np.lexsort((sv, su))
    su, sv, sw = su[o], sv[o], sw[o]
    nk = len(members)
    ids = np.arange(nk + 1, dtype=np.int64)
    w = np.concatenate([[0.0], vw[members].astype(np.float64)])
    return HostDag(ids, 0, su.astype(np.int32), sv.astype(np.int32), w, w, sw,
                   np.zeros(len(sw), dtype=np.int64))


def reference_recursive_parts(xadj: np.ndarray, adjncy: np.ndarray, adjwgt: np.ndarray,
                              vwgt: np.ndarray, k: int, tpwgts: Sequence[float], tol: float,
                              config: Optional[PartitionConfig] = None) -> np.ndarray:
    """int32 [n] part of every vertex: the reference heuristic applied recursively."""
    config = config or PartitionConfig(imbalance_tolerance=tol)
    n = len(vwgt)
    part = np.zeros(n, dtype=np.int32)
    eu, ev, ew = _undirected_edges(xadj, adjncy, adjwgt)
    cum = np.concatenate([[0.0], np.cumsum(np.asarray(tpwgts, dtype=np.float64))])
    todo: List[Tuple[int, int, np.ndarray]] = [(0, k, np.arange(n, dtype=np.int64))]
    dev = _native.device()
    R = config.restarts + 1
    while todo:
        split = [(p0, p1, m) for p0, p1, m in todo if p1 - p0 >= 2 and len(m) > 0]
        todo = []
        if not split:
            break
        hosts, work = [], []
        for p0, p1, m in split:
            pm = p0 + (p1 - p0) // 2
            ta, tb = cum[pm] - cum[p0], cum[p1] - cum[pm]
            r_cpu = ta / (ta + tb)
            w = vwgt[m].astype(np.float64)
            if r_cpu <= 0.0 or r_cpu >= 1.0 or not w.any():  # degenerate (partition.py:271-274)
                part[m] = p0 if r_cpu >= 1.0 else pm
                todo += [(p0, pm, m if r_cpu >= 1.0 else m[:0]),
                         (pm, p1, m[:0] if r_cpu >= 1.0 else m)]
                continue
            hosts.append(_subgraph(m, eu, ev, ew, vwgt))
            work.append((p0, pm, p1, m, r_cpu, w))
        if not work:
            continue
        tb_ = TwoWayBatch(hosts, dev)
        orders = np.concatenate([start_orders(w, config).reshape(-1) for *_, w in work])
        weights = torch.from_numpy(np.concatenate([w for *_, w in work])).to(dev)
        r = torch.tensor([x[4] for x in work], dtype=torch.float64, device=dev)
        assign, cut, err, status = _native.fm2_batch(tb_, weights, r, config.imbalance_tolerance,
                                                     torch.from_numpy(orders).to(dev), R)
        assign, cut, err = assign.cpu().numpy(), cut.cpu().numpy(), err.cpu().numpy()
        for b, (p0, pm, p1, m, _, w) in enumerate(work):
            nb = len(w)
            rows = assign[R * tb_.node_off_h[b]: R * tb_.node_off_h[b] + R * nb].reshape(R, nb)
            best = None
            for o in range(R):  # partition.py:291-294
                key = (not bool(err[b, o] <= config.imbalance_tolerance), float(cut[b, o]),
                       float(err[b, o]), tuple(rows[o].tolist()))
                if best is None or key < best[0]:
                    best = (key, o)
            side = rows[best[1]]
            left, right = m[side == 0], m[side != 0]
            part[left] = p0
            part[right] = pm
            todo += [(p0, pm, left), (pm, p1, right)]
    return part


def reference_recursive_start(ug, k: int, tpwgts: Sequence[float], tol: float) -> torch.Tensor:
    """``reference_recursive_parts`` of a ``kway.UGraph``, as a device int32 [1, n] start."""
    xadj = ug.xadj.cpu().numpy()
    adjncy = ug.adjncy.cpu().numpy()
    adjwgt = ug.adjwgt.cpu().numpy()
    vwgt = ug.vwgt.cpu().numpy()
    p = reference_recursive_parts(xadj, adjncy, adjwgt, vwgt, k, tpwgts, tol)
    return torch.from_numpy(p).to(ug.xadj.device).unsqueeze(0).contiguous()
