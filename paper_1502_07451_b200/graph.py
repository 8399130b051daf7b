"""Weighted task-DAG object model (drop-in mirror of ``hetsched.graph``).

The object model (``KernelNode``/``DataEdge``/``TaskGraph``) keeps the reference
names, fields and error behaviour so callers of ``hetsched`` can switch
packages. Heavy lifting never happens on these Python objects: every graph is
lowered once to a device-resident CSR (``paper_1502_07451_b200.csr``) and the
hot-path functions (evaluate, partition, simulate, critical path, weight
totals) run as sm_100a kernels on that CSR.

Reference: /root/reference/pkg/src/hetsched/graph.py (cited per symbol).
"""
from __future__ import annotations

from dataclasses import dataclass, replace
from typing import Dict, Iterable, List, Optional, Tuple

SOURCE_KIND = "SOURCE"
ROOT_ID = 0
CPU = "CPU"
GPU = "GPU"


class GraphError(Exception):
    """graph.py:17"""


class CycleError(GraphError):
    """graph.py:21-25 — carries the smallest id left with unresolved inputs."""

    def __init__(self, member: int):
        super().__init__(f"graph contains a cycle through node {member}")
        self.member = member


class InfeasibleGraphError(GraphError):
    """graph.py:27"""


@dataclass(frozen=True)
class KernelNode:
    """graph.py:31-39"""
    id: int
    kind: str
    size: int
    weight_cpu: float = 0.0
    weight_gpu: float = 0.0
    attrs: Tuple[Tuple[str, str], ...] = ()


@dataclass(frozen=True)
class DataEdge:
    """graph.py:42-48"""
    src: int
    dst: int
    bytes: int = 0
    weight_xfer: float = 0.0
    attrs: Tuple[Tuple[str, str], ...] = ()


class TaskGraph:
    """Immutable weighted DAG; node ``root`` is the zero-weight SOURCE.

    Mirrors graph.py:51-110: a later duplicate node/edge replaces the earlier
    one (and is recorded for ``validate``); successor and predecessor lists are
    kept ascending. The lowered device CSR is cached on the instance
    (``_csr_cache``) because the graph is immutable.
    """

    def __init__(self, nodes: Iterable[KernelNode], edges: Iterable[DataEdge],
                 root: int = ROOT_ID, name: str = "task"):
        self.name = name
        self.root = root
        self.nodes: Dict[int, KernelNode] = {}
        self.edges: Dict[Tuple[int, int], DataEdge] = {}
        self._duplicate_ids: List[int] = []
        self._duplicate_edges: List[Tuple[int, int]] = []
        for node in nodes:
            if node.id in self.nodes:
                self._duplicate_ids.append(node.id)
            self.nodes[node.id] = node
        for edge in edges:
            key = (edge.src, edge.dst)
            if key in self.edges:
                self._duplicate_edges.append(key)
            self.edges[key] = edge
        succ: Dict[int, List[int]] = {i: [] for i in self.nodes}
        pred: Dict[int, List[int]] = {i: [] for i in self.nodes}
        for (u, v) in self.edges:
            if u in succ and v in pred:
                succ[u].append(v)
                pred[v].append(u)
        for table in (succ, pred):
            for lst in table.values():
                lst.sort()
        self._succ = succ
        self._pred = pred
        self._csr_cache = None

    # -- queries (graph.py:85-110) -------------------------------------
    def successors(self, nid: int) -> List[int]:
        return self._succ.get(nid, [])

    def predecessors(self, nid: int) -> List[int]:
        return self._pred.get(nid, [])

    def in_edges(self, nid: int) -> List[DataEdge]:
        return [self.edges[(u, nid)] for u in self.predecessors(nid)]

    def kernel_ids(self) -> List[int]:
        return sorted(i for i in self.nodes if i != self.root)

    def n_kernels(self) -> int:
        return len(self.nodes) - (1 if self.root in self.nodes else 0)

    def inter_kernel_edges(self) -> List[DataEdge]:
        return [e for (u, _), e in sorted(self.edges.items()) if u != self.root]

    def replace_nodes(self, nodes: Iterable[KernelNode],
                      edges: Optional[Iterable[DataEdge]] = None) -> "TaskGraph":
        return TaskGraph(nodes, self.edges.values() if edges is None else edges,
                         root=self.root, name=self.name)

    def structurally_equal(self, other: "TaskGraph") -> bool:
        return (self.root == other.root and self.nodes == other.nodes
                and self.edges == other.edges)

    # -- device lowering ------------------------------------------------
    def csr(self):
        """Device CSR of this graph (built once, cached; see csr.py)."""
        if self._csr_cache is None:
            from .csr import DagCSR
            self._csr_cache = DagCSR.from_taskgraph(self)
        return self._csr_cache


def validate(graph: TaskGraph) -> List[str]:
    """All invariant violations, in the reference's message order (graph.py:113-150).

    The order matters: ``simulate`` reports ``problems[0]``.
    """
    out: List[str] = [f"duplicate node id {i}" for i in graph._duplicate_ids]
    out += [f"duplicate edge ({u}, {v})" for (u, v) in graph._duplicate_edges]
    root_node = graph.nodes.get(graph.root)
    if root_node is None:
        out.append(f"root node {graph.root} missing")
    elif root_node.kind != SOURCE_KIND:
        out.append(f"root node {graph.root} is not kind {SOURCE_KIND}")
    for node in graph.nodes.values():
        if node.weight_cpu < 0 or node.weight_gpu < 0:
            out.append(f"node {node.id} has negative weight")
        if node.kind == SOURCE_KIND and (node.weight_cpu != 0 or node.weight_gpu != 0):
            out.append(f"{SOURCE_KIND} node {node.id} must have zero weights")
    for (u, v), e in sorted(graph.edges.items()):
        if u == v:
            out.append(f"self-loop on node {u}")
        for end in (u, v):
            if end not in graph.nodes:
                out.append(f"edge ({u}, {v}) references unknown node {end}")
        if e.weight_xfer < 0:
            out.append(f"edge ({u}, {v}) has negative transfer weight")
        if e.bytes < 0:
            out.append(f"edge ({u}, {v}) has negative byte count")
    try:
        topological_order(graph)
    except CycleError as exc:
        out.append(f"cycle through node {exc.member}")
    if root_node is not None:
        out += [f"initial kernel {i} has no edge from root"
                for i in graph.nodes if i != graph.root and not graph.predecessors(i)]
    return out


def topological_order(graph: TaskGraph) -> List[int]:
    """Lexicographically smallest topological order (graph.py:153-172).

    Kahn's algorithm with an id min-heap, run on the device
    (``hs_topological_order``: the identity when every edge points to a
    larger id, batched heap rounds otherwise); on a cycle raises CycleError
    with the smallest id whose in-degree never reached zero.
    """
    if not graph.nodes:
        return []
    from . import _native
    csr = graph.csr()
    order, count, stuck, _ = _native.topological_order(csr)
    if count != csr.n:
        raise CycleError(int(csr.ids[stuck]))
    return csr.ids[order.cpu().numpy()].tolist()


def attach_weights(graph: TaskGraph, model) -> TaskGraph:
    """Copy of ``graph`` with node/edge weights from ``model`` (graph.py:308-324).

    The weights are computed on the device (``hs_attach_weights``, one entry
    per distinct (kind, size) pair: the synthetic closed forms per node, any
    other model read once per pair); the root (or any SOURCE node) is forced
    to zero weight. The first node in the graph's node order without a cost
    entry raises GraphError with the model's own message, a negative byte
    count the model's CostModelError, as the reference does.
    """
    import numpy as np
    import torch
    from . import _native
    from .costs import device_weights
    nodes = list(graph.nodes.values())
    edges = list(graph.edges.values())
    keys, index = [], {}
    pair = np.empty(len(nodes), dtype=np.int32)
    size = np.empty(len(nodes), dtype=np.int64)
    for r, node in enumerate(nodes):
        key = None if (node.id == graph.root or node.kind == SOURCE_KIND) else (node.kind, node.size)
        if key not in index:
            index[key] = len(keys)
            keys.append(key)
        pair[r] = index[key]
        size[r] = node.size if -2 ** 63 <= node.size < 2 ** 63 else 0
    dev = _native.device()
    t = lambda a: torch.from_numpy(a).to(dev)  # noqa: E731
    nbytes = np.fromiter((e.bytes for e in edges), dtype=np.int64, count=len(edges))
    w_cpu, w_gpu, w_xfer, bad_node, bad_edge = device_weights(
        model, keys, t(pair), t(size), t(nbytes), rank=None, device=dev)
    if bad_node >= 0:
        node = nodes[bad_node]
        try:
            model.kernel_time(node.kind, node.size, CPU)
            model.kernel_time(node.kind, node.size, GPU)
        except Exception as exc:
            raise GraphError(f"no cost entry for kernel {node.id} "
                             f"({node.kind}, {node.size}): {exc}") from exc
        raise GraphError(f"no cost entry for kernel {node.id} ({node.kind}, {node.size})")
    if bad_edge >= 0:
        model.transfer_time(edges[bad_edge].bytes)  # raises the model's CostModelError
    wc, wg, wx = (x.cpu().numpy().tolist() for x in (w_cpu, w_gpu, w_xfer))
    new_nodes = [replace(node, weight_cpu=wc[r], weight_gpu=wg[r]) for r, node in enumerate(nodes)]
    new_edges = [replace(e, weight_xfer=wx[i]) for i, e in enumerate(edges)]
    return graph.replace_nodes(new_nodes, new_edges)


def total_weights(graph: TaskGraph) -> Tuple[float, float, float]:
    """Correctly rounded (fsum) totals of w_cpu, w_gpu, w_xfer (graph.py:327-332).

    Runs on the device: an exact fixed-point superaccumulator rounded once,
    which is what ``math.fsum`` returns.
    """
    from . import _native
    csr = graph.csr()
    return _native.exact_totals(csr, include_root=True)


# generate_random_dag lives in gen.py (input synthesis); re-exported here so
# ``from ...graph import generate_random_dag`` keeps working.
from .gen import generate_random_dag  # noqa: E402,F401
