"""Input synthesis: task DAG generators.

* ``generate_random_dag`` — the reference's layered two-input generator
  (graph.py:180-305), restated with the same ``random.Random`` draw sequence so
  the graphs are identical, but in O(n + E) instead of the reference's O(n·E)
  (graph.py:259 ``slot_kernels.count``, graph.py:299-301 root-wiring scan).
* ``cholesky_dag`` — the right-looking tiled-Cholesky task DAG.
* ``layered_dag`` (in ``csr.py``/``_native``) — the device generator for the
  100k/1M and 10M/100M layered fan-in DAGs of configs 2 and 4.
"""
from __future__ import annotations

import math
import random
from collections import Counter
from typing import Dict, List, Optional, Tuple


def _split_even(n: int, parts: int) -> List[int]:
    q, r = divmod(n, parts)
    return [q + 1 if i < r else q for i in range(parts)]


def generate_random_dag(n_kernels: int, n_edges: int, kind: str, size: int,
                        seed: int, layers: Optional[int] = None,
                        count_root: bool = False):
    """Layered random DAG of two-input kernels; identical output to graph.py:180-305.

    The random stream is consumed in exactly the reference order: one
    ``sample`` over the input slots (only when they are not all used), one
    ``sample`` of predecessors per kernel in id order, one ``sample`` of
    surplus sink pairs.
    """
    from .graph import (DataEdge, InfeasibleGraphError, KernelNode, ROOT_ID,
                        SOURCE_KIND, TaskGraph)
    rng = random.Random(seed)
    payload = size * size * 4
    n_real = n_kernels - 1 if count_root else n_kernels
    if n_real < 1:
        raise InfeasibleGraphError("need at least one kernel")
    n_layers = min(layers if layers else max(1, math.ceil(math.sqrt(n_real))), n_real)
    sizes = _split_even(n_real, n_layers)

    # layer li holds ids [first[li], first[li] + sizes[li]); everything below
    # first[li] is "earlier" for that layer
    first = [1]
    for s in sizes:
        first.append(first[-1] + s)
    last_lo, last_hi = first[-2], first[-1]

    # two input slots per kernel past layer 0 (one if only one earlier kernel)
    slot_kernels: List[int] = []
    for li in range(1, n_layers):
        reps = min(2, first[li] - 1)
        for k in range(first[li], first[li + 1]):
            slot_kernels.extend([k] * reps)
    base_capacity = len(slot_kernels)
    n_earlier_last = last_lo - 1

    if count_root:
        inter_target = n_edges - sizes[0]
        min_inter = n_real - sizes[0]
        if inter_target < min_inter:
            raise InfeasibleGraphError(
                f"{n_edges} total edges cannot cover {n_real} kernels")
    else:
        inter_target = n_edges
        min_inter = 0
    overflow = (sizes[-1] * max(0, n_earlier_last - 2)) if n_layers > 1 else 0
    if inter_target > base_capacity + overflow:
        raise InfeasibleGraphError(
            f"{n_edges} edges infeasible for {n_real} two-input kernels")

    if inter_target >= base_capacity:
        counts: Dict[int, int] = Counter(slot_kernels)
        extra = inter_target - base_capacity
    else:
        if min_inter:
            mandatory = sorted(set(slot_kernels))
            # drop the first occurrence of each kernel (list.remove semantics)
            seen = set()
            pool = []
            for k in slot_kernels:
                if k in seen:
                    pool.append(k)
                else:
                    seen.add(k)
            picks = mandatory + rng.sample(pool, inter_target - len(mandatory))
        else:
            picks = rng.sample(slot_kernels, inter_target)
        counts = Counter(picks)
        extra = 0

    edges: List = []
    used = set()
    for li in range(1, n_layers):
        earlier = range(1, first[li])
        for k in range(first[li], first[li + 1]):
            c = counts.get(k, 0)
            if c:
                for u in rng.sample(earlier, c):
                    edges.append(DataEdge(u, k, bytes=payload))
                    used.add((u, k))
    if extra:
        candidates = [(u, k) for k in range(last_lo, last_hi)
                      for u in range(1, last_lo) if (u, k) not in used]
        if extra > len(candidates):
            raise InfeasibleGraphError(
                f"{n_edges} edges infeasible for {n_real} two-input kernels")
        for (u, k) in rng.sample(candidates, extra):
            edges.append(DataEdge(u, k, bytes=payload))
            used.add((u, k))
    fed = {k for (_, k) in used}
    for k in range(1, last_hi):
        if k not in fed:
            edges.append(DataEdge(ROOT_ID, k, bytes=payload))
    nodes = [KernelNode(ROOT_ID, SOURCE_KIND, 0)]
    nodes += [KernelNode(k, kind, size) for k in range(1, last_hi)]
    return TaskGraph(nodes, edges)


def random_dag_shape(n_kernels: int, n_edges: int, layers: Optional[int] = None,
                     count_root: bool = False) -> dict:
    """The seed-independent part of generate_random_dag (graph.py:195-252):
    layer bounds, slot capacity, targets; raises the reference's
    InfeasibleGraphError exactly where generate_random_dag does."""
    from .graph import InfeasibleGraphError
    n_real = n_kernels - 1 if count_root else n_kernels
    if n_real < 1:
        raise InfeasibleGraphError("need at least one kernel")
    n_layers = min(layers if layers else max(1, math.ceil(math.sqrt(n_real))), n_real)
    sizes = _split_even(n_real, n_layers)
    first = [1]
    for s in sizes:
        first.append(first[-1] + s)
    base_capacity = sum(min(2, first[li] - 1) * sizes[li] for li in range(1, n_layers))
    n_earlier_last = first[-2] - 1
    if count_root:
        inter_target = n_edges - sizes[0]
        min_inter = n_real - sizes[0]
        if inter_target < min_inter:
            raise InfeasibleGraphError(f"{n_edges} total edges cannot cover {n_real} kernels")
    else:
        inter_target, min_inter = n_edges, 0
    overflow = (sizes[-1] * max(0, n_earlier_last - 2)) if n_layers > 1 else 0
    if inter_target > base_capacity + overflow:
        raise InfeasibleGraphError(f"{n_edges} edges infeasible for {n_real} two-input kernels")
    if inter_target >= base_capacity:
        mode, extra = 0, inter_target - base_capacity
    else:
        mode, extra = (2 if min_inter else 1), 0
    # (the reference's second check, extra > unused sink pairs, graph.py:288,
    # cannot fire past the first: with every slot used each last-layer kernel
    # holds min(2, earlier) inputs, so the unused pairs are exactly the overflow)
    n_cand = sizes[-1] * n_earlier_last if n_layers > 1 else 0
    return {"n_real": n_real, "n_layers": n_layers, "first": first,
            "base_capacity": base_capacity, "inter_target": inter_target, "extra": extra,
            "mode": mode, "pop_cap": 2 * max(base_capacity, n_real, n_cand) + 2,
            "edge_cap": inter_target + n_real}


def generate_random_dag_batch(n_kernels: int, n_edges: int, kind: str, size: int, seeds,
                              model=None, layers: Optional[int] = None,
                              count_root: bool = False):
    """generate_random_dag(n_kernels, n_edges, kind, size, seed) for every seed,
    built on the device (csrc/rgen.cu: CPython's Random per graph, same draw
    order) and weighted by ``model`` (default SyntheticCostModel, the
    attach_weights of configs 1 and 5) on the device: a DagBatch, graph b
    identical to attach_weights(generate_random_dag(..., seeds[b]), model)."""
    import numpy as np
    import torch
    from . import _native
    from .costs import SyntheticCostModel, device_weights
    from .csr import DagBatch
    model = model or SyntheticCostModel()
    shape = random_dag_shape(n_kernels, n_edges, layers, count_root)
    seeds = [int(x) for x in seeds]
    if any(abs(x) >= 2 ** 63 for x in seeds):
        raise ValueError("seeds must fit in 64 bits")
    dev = _native.device()
    sd = torch.tensor(seeds, dtype=torch.int64, device=dev)
    n = shape["n_real"] + 1
    m, out_ptr, out_dst, in_ptr, in_src, in_eid = _native.random_dag_batch(sd, shape, n)
    b = len(seeds)
    node_counts = np.full(b, n, dtype=np.int64)
    # weights: the root zero, every kernel (kind, size); every edge one size^2 fp32 matrix
    pair = torch.zeros(b * n, dtype=torch.int32, device=dev)
    pair[::n] = 1
    sizes = torch.full((b * n,), size, dtype=torch.int64, device=dev)
    nbytes = torch.full((int(m.sum()),), size * size * 4, dtype=torch.int64, device=dev)
    w_cpu, w_gpu, w_xfer, bad_node, bad_edge = device_weights(model, [(kind, size), None], pair,
                                                             sizes, nbytes, device=dev)
    if bad_node >= 0:
        from .graph import GraphError
        try:
            model.kernel_time(kind, size, "CPU")
            model.kernel_time(kind, size, "GPU")
        except Exception as exc:
            raise GraphError(f"no cost entry for kernel 1 ({kind}, {size}): {exc}") from exc
    root = torch.zeros(b, dtype=torch.int32, device=dev)
    return DagBatch.from_device(node_counts, m, root, out_ptr, out_dst, in_ptr, in_src, in_eid,
                                w_cpu, w_gpu, w_xfer, nbytes)


class RandomDagFactory:
    """``seed -> attach_weights(generate_random_dag(n, m, kind, size, seed), model)``.

    Called with a seed it builds the TaskGraph exactly as the reference does
    (graph_factory of sim.compare); ``compare`` recognises it and generates
    all iterations at once on the device instead (``batch``)."""

    def __init__(self, n_kernels: int, n_edges: int, kind: str = "MA", size: int = 1024,
                 model=None, layers: Optional[int] = None, count_root: bool = False):
        self.n_kernels, self.n_edges, self.kind, self.size = n_kernels, n_edges, kind, size
        self.model, self.layers, self.count_root = model, layers, count_root

    def __call__(self, seed: int):
        from .costs import SyntheticCostModel
        from .graph import attach_weights
        g = generate_random_dag(self.n_kernels, self.n_edges, self.kind, self.size, seed,
                                self.layers, self.count_root)
        return attach_weights(g, self.model or SyntheticCostModel())

    def batch(self, seeds):
        return generate_random_dag_batch(self.n_kernels, self.n_edges, self.kind, self.size,
                                         seeds, self.model, self.layers, self.count_root)


def cholesky_tasks(tiles: int) -> Tuple[List[Tuple[str, Tuple[int, ...]]], List[Tuple[int, int]]]:
    """Right-looking tiled Cholesky task list and last-writer dependencies.

    Returns (tasks, deps): tasks[t-1] = (kind, (i, j, k)) for task id t
    (1-based, creation order), deps = sorted unique (producer, consumer).
    Construction follows SURVEY.md Appendix D; T=8 gives 120 tasks/252 edges,
    T=64 gives 45,760 tasks/131,040 edges.
    """
    tasks: List[Tuple[str, Tuple[int, ...]]] = []
    last: Dict[Tuple[int, int], int] = {}
    deps = set()

    def add(kind, key, out_tile, inputs):
        tasks.append((kind, key))
        tid = len(tasks)
        for src in inputs:
            if src:
                deps.add((src, tid))
        last[out_tile] = tid
        return tid

    trsm_of: Dict[Tuple[int, int], int] = {}
    for k in range(tiles):
        potrf = add("POTRF", (k, k, k), (k, k), [last.get((k, k), 0)])
        for i in range(k + 1, tiles):
            trsm_of[(i, k)] = add("TRSM", (i, k, k), (i, k), [potrf, last.get((i, k), 0)])
        for i in range(k + 1, tiles):
            add("SYRK", (i, i, k), (i, i), [trsm_of[(i, k)], last.get((i, i), 0)])
            for j in range(k + 1, i):
                add("GEMM", (i, j, k), (i, j),
                    [trsm_of[(i, k)], trsm_of[(j, k)], last.get((i, j), 0)])
    return tasks, sorted(deps)


def cholesky_dag(tiles: int, block: int = 512, model=None):
    """Tiled-Cholesky TaskGraph (kinds POTRF/TRSM/SYRK/GEMM, size=block).

    Edge bytes are one fp64 tile (block²·8). The root feeds every task
    without a producer, as ``parse_dot`` does for in-degree-0 kernels
    (graphio.py:192-198). With ``model`` the weights are attached.
    """
    from .graph import DataEdge, KernelNode, ROOT_ID, SOURCE_KIND, TaskGraph, attach_weights
    tasks, deps = cholesky_tasks(tiles)
    tile_bytes = block * block * 8
    nodes = [KernelNode(ROOT_ID, SOURCE_KIND, 0)]
    nodes += [KernelNode(t + 1, kind, block) for t, (kind, _) in enumerate(tasks)]
    has_pred = {v for (_, v) in deps}
    edges = [DataEdge(u, v, bytes=tile_bytes) for (u, v) in deps]
    edges += [DataEdge(ROOT_ID, t, bytes=tile_bytes)
              for t in range(1, len(tasks) + 1) if t not in has_pred]
    g = TaskGraph(nodes, edges, name="cholesky")
    return attach_weights(g, model) if model is not None else g
