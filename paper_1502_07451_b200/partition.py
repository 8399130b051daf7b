"""Balanced min-cut partitioning (drop-in mirror of ``hetsched.partition``).

* ``partition_heuristic`` / ``fm_refine`` / ``brute_force_partition`` /
  ``evaluate`` keep the reference's 2-way semantics bit for bit: the greedy
  init, balance repair and FM passes run on the device (csrc/fm2.cu), one CTA
  per start order, with the reference's fp64 arithmetic and tie-breaking.
* ``partition_kway`` is the multilevel k-way partitioner (csrc/kway.cu) for
  graphs far beyond what FM can handle (configs 2-4).

Reference: /root/reference/pkg/src/hetsched/partition.py (cited per symbol).
"""
from __future__ import annotations

import random
from dataclasses import dataclass
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np
import torch

from . import _native
from .costs import PartitionTargets
from .graph import CPU, GPU, TaskGraph


class PartitionError(Exception):
    """partition.py:17"""


@dataclass
class PartitionConfig:
    """partition.py:21-34"""
    node_weight_source: str = GPU
    imbalance_tolerance: float = 0.03
    restarts: int = 8
    seed: int = 0

    def __post_init__(self):
        if self.node_weight_source not in (CPU, GPU):
            raise PartitionError(f"bad node weight source {self.node_weight_source!r}")
        if not 0.0 <= self.imbalance_tolerance < 1.0:
            raise PartitionError("imbalance tolerance must be in [0, 1)")
        if self.restarts < 1:
            raise PartitionError("restarts must be >= 1")


@dataclass
class Partition:
    """partition.py:37-45"""
    assignment: Dict[int, str]
    edge_cut: float
    balance_error: float
    targets: PartitionTargets
    node_weight_source: str = GPU
    feasible: bool = True
    side_weights: Tuple[float, float] = (0.0, 0.0)


def _node_weight(node, source: str) -> float:
    return node.weight_gpu if source == GPU else node.weight_cpu


def _weights(csr, source: str) -> torch.Tensor:
    """Per-kernel weights (kernel position order) on the device."""
    w = csr.w_gpu if source == GPU else csr.w_cpu
    return torch.cat([w[:csr.root], w[csr.root + 1:]]).contiguous()


def _kernel_ids(csr) -> np.ndarray:
    ids = csr.host.ids
    return np.concatenate([ids[:csr.root], ids[csr.root + 1:]])


def _assignment_array(csr, assignment: Dict[int, str]) -> np.ndarray:
    ids = _kernel_ids(csr)
    return np.fromiter((0 if assignment[int(i)] == CPU else 1 for i in ids),
                       dtype=np.int8, count=len(ids))


def _assignment_dict(csr, arr: np.ndarray) -> Dict[int, str]:
    ids = _kernel_ids(csr)
    return {int(i): (CPU if a == 0 else GPU) for i, a in zip(ids, arr)}


def _evaluate_arrays(graph: TaskGraph, parts: np.ndarray, source: str):
    csr = graph.csr()
    dev = csr.device
    t = torch.from_numpy(np.ascontiguousarray(parts.reshape(-1, csr.n_kernels))).to(dev)
    cut, cpu_w, total = _native.evaluate2(csr, t, 1 if source == GPU else 0, 0)
    return cut.cpu().numpy(), cpu_w.cpu().numpy(), total.cpu().numpy()


def evaluate(graph: TaskGraph, partition: Partition) -> Tuple[float, float, Tuple[float, float]]:
    """Cut, balance error and side weights recomputed on the device (partition.py:60-73).

    Sums run in the reference's order with CPython's float ``sum`` semantics
    (K2 mode 0), so the result is bit-identical to the reference's.
    """
    ids = graph.kernel_ids()
    if set(partition.assignment) != set(ids):
        raise PartitionError("partition does not cover exactly the non-root kernels")
    csr = graph.csr()
    arr = _assignment_array(csr, partition.assignment)
    cut, cpu_w, total = _evaluate_arrays(graph, arr, partition.node_weight_source)
    cut, cpu_w, total = float(cut[0]), float(cpu_w[0]), float(total[0])
    if total == 0:
        raise PartitionError("zero total node weight; attach weights first")
    err = abs(cpu_w / total - partition.targets.r_cpu)
    return cut, err, (cpu_w, total - cpu_w)


def _finish(graph: TaskGraph, assignment: Dict[int, str], targets: PartitionTargets,
            source: str, tolerance: float) -> Partition:
    """partition.py:76-84 — shares evaluate()'s device path."""
    p = Partition(dict(assignment), 0.0, 0.0, targets, source)
    cut, err, sides = evaluate(graph, p)
    p.edge_cut, p.balance_error, p.side_weights = cut, err, sides
    p.feasible = err <= tolerance
    return p


def brute_force_partition(graph: TaskGraph, targets: PartitionTargets, tolerance: float,
                          node_weight_source: str = GPU) -> Partition:
    """Exhaustive minimum-cut oracle for n <= 20 (partition.py:87-134), 2^n masks on device."""
    ids = graph.kernel_ids()
    n = len(ids)
    if n == 0:
        raise PartitionError("graph has no non-root kernels")
    if n > 20:
        raise PartitionError(f"brute force refuses {n} kernels (limit 20)")
    csr = graph.csr()
    tw = csr.twoway()
    w = _weights(csr, node_weight_source)
    try:
        mask, _ = _native.brute2(n, w, targets.r_cpu, tolerance, tw.edge_u, tw.edge_v,
                                 tw.edge_w)
    except _native.NativeError as exc:
        raise PartitionError(exc.message) from exc
    arr = np.array([(mask >> (n - 1 - k)) & 1 for k in range(n)], dtype=np.int8)
    return _finish(graph, _assignment_dict(csr, arr), targets, node_weight_source, tolerance)


def _run_fm(graph: TaskGraph, targets: PartitionTargets, config: PartitionConfig,
            orders: Optional[np.ndarray], start: Optional[np.ndarray]):
    csr = graph.csr()
    tw = csr.twoway()
    dev = csr.device
    w = _weights(csr, config.node_weight_source)
    o = torch.from_numpy(orders.astype(np.int32)).to(dev) if orders is not None else None
    s = torch.from_numpy(start.astype(np.int8)).to(dev) if start is not None else None
    if o is None:
        dummy = torch.zeros(1, csr.n_kernels, dtype=torch.int32, device=dev)
    try:
        assign, cut, err = _native.fm2(tw, tw.edge_w, tw.edge_u, tw.edge_v, w, targets.r_cpu,
                                       config.imbalance_tolerance,
                                       o if o is not None else dummy, s)
    except _native.NativeError as exc:
        raise PartitionError(exc.message) from exc
    return assign.cpu().numpy(), cut.cpu().numpy(), err.cpu().numpy()


def fm_refine(graph: TaskGraph, partition: Partition, targets: PartitionTargets,
              config: PartitionConfig) -> Partition:
    """FM passes from ``partition`` (partition.py:137-220), one CTA on the device."""
    csr = graph.csr()
    start = _assignment_array(csr, partition.assignment)
    assign, _, _ = _run_fm(graph, targets, config, None, start)
    return _finish(graph, _assignment_dict(csr, assign[0]), targets,
                   config.node_weight_source, config.imbalance_tolerance)


def start_orders(weights: np.ndarray, config: PartitionConfig) -> np.ndarray:
    """The reference's start orders (partition.py:280-285), as kernel positions.

    Order 0: descending weight, stable. Order 1+r: ``random.Random(seed *
    1_000_003 + r).shuffle`` of the id list — drawn with CPython's own
    generator so the permutations are identical.
    """
    n = len(weights)
    orders = np.empty((config.restarts + 1, n), dtype=np.int32)
    orders[0] = np.argsort(-weights, kind="stable")
    for r in range(config.restarts):
        perm = list(range(n))
        random.Random(config.seed * 1_000_003 + r).shuffle(perm)
        orders[r + 1] = perm
    return orders


def partition_heuristic(graph: TaskGraph, targets: PartitionTargets,
                        config: Optional[PartitionConfig] = None) -> Partition:
    """Multi-restart greedy + FM, deterministic per seed (partition.py:258-295).

    All 1 + restarts start orders are refined concurrently, one CTA each;
    the winner is the reference's minimum of (not feasible, cut, err, lex).
    """
    config = config or PartitionConfig()
    ids = graph.kernel_ids()
    if not ids:
        raise PartitionError("graph has no non-root kernels")
    source, tol = config.node_weight_source, config.imbalance_tolerance
    csr = graph.csr()
    w_host = np.array([_node_weight(graph.nodes[i], source) for i in ids], dtype=np.float64)
    if not np.any(w_host):
        raise PartitionError("zero total node weight; attach weights first")
    if targets.r_cpu == 0.0 or targets.r_cpu == 1.0:
        side = GPU if targets.r_cpu == 0.0 else CPU
        return _finish(graph, {i: side for i in ids}, targets, source, tol)
    orders = start_orders(w_host, config)
    assign, cut, err = _run_fm(graph, targets, config, orders, None)
    best = None
    for k in range(len(orders)):
        key = (not bool(err[k] <= tol), float(cut[k]), float(err[k]), tuple(assign[k].tolist()))
        if best is None or key < best[0]:
            best = (key, k)
    return _finish(graph, _assignment_dict(csr, assign[best[1]]), targets, source, tol)


_ORDER_CACHE: Dict[Tuple[int, int, int], np.ndarray] = {}


def _shuffles(n: int, config: PartitionConfig) -> np.ndarray:
    """The restart permutations depend only on (n, seed, restarts): cached."""
    key = (n, config.seed, config.restarts)
    if key not in _ORDER_CACHE:
        out = np.empty((config.restarts, n), dtype=np.int32)
        for r in range(config.restarts):
            perm = list(range(n))
            random.Random(config.seed * 1_000_003 + r).shuffle(perm)
            out[r] = perm
        _ORDER_CACHE[key] = out
    return _ORDER_CACHE[key]


def partition_heuristic_batch(graphs: Sequence[TaskGraph], targets: Sequence[PartitionTargets],
                              config: Optional[PartitionConfig] = None) -> List[Dict[int, str]]:
    """``partition_heuristic`` for many graphs in one launch; returns the assignments.

    Same semantics per graph (partition.py:258-295): degenerate targets
    short-circuit, otherwise 1 + restarts start orders refined by FM on the
    device (one CTA per graph x order), winner by (not feasible, cut, err, lex).
    """
    config = config or PartitionConfig()
    source = config.node_weight_source
    hosts, ws = [], []
    for g in graphs:
        ids = g.kernel_ids()
        if not ids:
            raise PartitionError("graph has no non-root kernels")
        hosts.append(g.csr().host)
        ws.append(np.array([_node_weight(g.nodes[i], source) for i in ids], dtype=np.float64))
    rows = partition_rows_batch(hosts, ws, [t.r_cpu for t in targets], config)
    return [_assignment_dict(g.csr(), r) for g, r in zip(graphs, rows)]


def partition_rows_batch(hosts, ws, r_cpu, config: PartitionConfig) -> List[np.ndarray]:
    """The device part of partition_heuristic_batch on HostDags: per graph
    the winning assignment as an int8 row over its kernels (0 CPU, 1 GPU).
    ws[b] = kernel weights (kernel position order), r_cpu[b] = target."""
    from .csr import TwoWayBatch
    tol = config.imbalance_tolerance
    out: List[Optional[np.ndarray]] = [None] * len(hosts)
    work = []
    for gi, (h, w, r) in enumerate(zip(hosts, ws, r_cpu)):
        if not len(w):
            raise PartitionError("graph has no non-root kernels")
        if not np.any(w):
            raise PartitionError("zero total node weight; attach weights first")
        if r == 0.0 or r == 1.0:
            out[gi] = np.full(len(w), 1 if r == 0.0 else 0, dtype=np.int8)
        else:
            work.append((gi, h, r, w))
    if not work:
        return out
    R = config.restarts + 1
    tb = TwoWayBatch([h for _, h, _, _ in work])
    orders = []
    for _, _, _, w in work:
        o = np.empty((R, len(w)), dtype=np.int32)
        o[0] = np.argsort(-w, kind="stable")
        o[1:] = _shuffles(len(w), config)
        orders.append(o.reshape(-1))
    dev = tb.xadj.device
    weights = torch.from_numpy(np.concatenate([w for *_, w in work])).to(dev)
    rt = torch.tensor([r for _, _, r, _ in work], dtype=torch.float64, device=dev)
    ordt = torch.from_numpy(np.concatenate(orders)).to(dev)
    assign, cut, err, status = _native.fm2_batch(tb, weights, rt, tol, ordt, R)
    if bool((status != 0).any()):
        raise PartitionError("zero total node weight; attach weights first")
    assign, cut, err = assign.cpu().numpy(), cut.cpu().numpy(), err.cpu().numpy()
    for b, (gi, _, _, w) in enumerate(work):
        n = len(w)
        rows = assign[R * tb.node_off_h[b]: R * tb.node_off_h[b] + R * n].reshape(R, n)
        best = None
        for k in range(R):
            key = (not bool(err[b, k] <= tol), float(cut[b, k]), float(err[b, k]),
                   tuple(rows[k].tolist()))
            if best is None or key < best[0]:
                best = (key, k)
        out[gi] = rows[best[1]].astype(np.int8)
    return out
    R = config.restarts + 1
    tb = TwoWayBatch([g.csr().host for _, g, _, _ in work])
    orders = []
    for _, g, _, w in work:
        o = np.empty((R, len(w)), dtype=np.int32)
        o[0] = np.argsort(-w, kind="stable")
        o[1:] = _shuffles(len(w), config)
        orders.append(o.reshape(-1))
    dev = tb.xadj.device
    weights = torch.from_numpy(np.concatenate([w for *_, w in work])).to(dev)
    r = torch.tensor([t.r_cpu for _, _, t, _ in work], dtype=torch.float64, device=dev)
    ordt = torch.from_numpy(np.concatenate(orders)).to(dev)
    assign, cut, err, status = _native.fm2_batch(tb, weights, r, tol, ordt, R)
    if bool((status != 0).any()):
        raise PartitionError("zero total node weight; attach weights first")
    assign, cut, err = assign.cpu().numpy(), cut.cpu().numpy(), err.cpu().numpy()
    for b, (gi, g, _, w) in enumerate(work):
        n = len(w)
        rows = assign[R * tb.node_off_h[b]: R * tb.node_off_h[b] + R * n].reshape(R, n)
        best = None
        for k in range(R):
            key = (not bool(err[b, k] <= tol), float(cut[b, k]), float(err[b, k]),
                   tuple(rows[k].tolist()))
            if best is None or key < best[0]:
                best = (key, k)
        out[gi] = _assignment_dict(g.csr(), rows[best[1]])
    return out
