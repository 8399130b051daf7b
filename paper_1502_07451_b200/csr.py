"""Device-resident CSR layouts of task DAGs (the HBM data layout of the hot path).

``DagCSR``  — one directed DAG: out-CSR sorted by (src, dst) (the reference's
              ``sorted(graph.edges)`` order), in-CSR with ascending sources
              (``graph.in_edges``, graph.py:89-90), fp64 node/edge weights,
              int64 byte counts. int64 row pointers, int32 indices.
``DagBatch`` — many small DAGs back to back (config 5's 4096 simulations).
``TwoWayGraph`` — the undirected kernel graph ``fm_refine`` builds
              (partition.py:153-158) with the reference's neighbour order, plus
              the inter-kernel edge list in sorted order, for the exact 2-way
              partitioner.

Host-side construction from ``TaskGraph`` objects is numpy; graphs generated
on the device (``layered``) never leave HBM.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np
import torch

from . import _native


def _csr_ptr(keys: np.ndarray, n: int) -> np.ndarray:
    ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(keys, minlength=n), out=ptr[1:])
    return ptr


@dataclass
class HostDag:
    """numpy arrays of one DAG in node-index space (see include/hetsched_b200.h)."""
    ids: np.ndarray        # int64 [n] original node ids, ascending
    root: int              # index of the root, -1 if absent
    src: np.ndarray        # int32 [m] sorted by (src, dst)
    dst: np.ndarray        # int32 [m]
    w_cpu: np.ndarray      # f64 [n]
    w_gpu: np.ndarray      # f64 [n]
    w_xfer: np.ndarray     # f64 [m]
    bytes: np.ndarray      # int64 [m]

    @property
    def n(self) -> int:
        return len(self.ids)

    @property
    def m(self) -> int:
        return len(self.src)

    def out_ptr(self) -> np.ndarray:
        return _csr_ptr(self.src, self.n)

    def in_order(self) -> np.ndarray:
        return np.lexsort((self.src, self.dst)).astype(np.int32)

    @classmethod
    def from_taskgraph(cls, graph) -> "HostDag":
        ids = np.array(sorted(graph.nodes), dtype=np.int64)
        index = {int(i): k for k, i in enumerate(ids)}
        items = sorted((index[u], index[v], e) for (u, v), e in graph.edges.items()
                       if u in index and v in index)
        m = len(items)
        src = np.fromiter((t[0] for t in items), dtype=np.int32, count=m)
        dst = np.fromiter((t[1] for t in items), dtype=np.int32, count=m)
        w_xfer = np.fromiter((t[2].weight_xfer for t in items), dtype=np.float64, count=m)
        nbytes = np.fromiter((t[2].bytes for t in items), dtype=np.int64, count=m)
        nodes = [graph.nodes[int(i)] for i in ids]
        w_cpu = np.fromiter((nd.weight_cpu for nd in nodes), dtype=np.float64, count=len(ids))
        w_gpu = np.fromiter((nd.weight_gpu for nd in nodes), dtype=np.float64, count=len(ids))
        root = index.get(graph.root, -1)
        return cls(ids, root, src, dst, w_cpu, w_gpu, w_xfer, nbytes)


class DagCSR:
    """Device CSR of one DAG; see module docstring."""

    def __init__(self, n: int, m: int, root: int, out_ptr, out_dst, in_ptr, in_src, in_eid,
                 w_cpu, w_gpu, w_xfer, nbytes, ids: Optional[np.ndarray] = None,
                 host: Optional[HostDag] = None):
        self.n, self.m, self.root = int(n), int(m), int(root)
        self.out_ptr, self.out_dst = out_ptr, out_dst
        self.in_ptr, self.in_src, self.in_eid = in_ptr, in_src, in_eid
        self.w_cpu, self.w_gpu, self.w_xfer, self.bytes = w_cpu, w_gpu, w_xfer, nbytes
        self.ids = ids
        self.host = host
        self.device = out_ptr.device
        self._struct = None
        self._twoway = None

    @classmethod
    def from_host(cls, h: HostDag, device=None) -> "DagCSR":
        dev = device or _native.device()
        order = h.in_order()
        t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
        return cls(h.n, h.m, h.root, t(h.out_ptr()), t(h.dst), t(_csr_ptr(h.dst, h.n)),
                   t(h.src[order]), t(order), t(h.w_cpu), t(h.w_gpu), t(h.w_xfer),
                   t(h.bytes), ids=h.ids, host=h)

    @classmethod
    def from_out_csr(cls, root: int, out_ptr: torch.Tensor, out_dst: torch.Tensor,
                     w_cpu=None, w_gpu=None, w_xfer=None, nbytes=None) -> "DagCSR":
        """DAG from its device out-CSR alone (edges sorted by (src, dst)); the
        in-CSR is built on the device (``hs_dag_transpose``)."""
        n, m = int(out_ptr.numel()) - 1, int(out_dst.numel())
        dev = out_ptr.device
        in_ptr = torch.empty(n + 1, dtype=torch.int64, device=dev)
        in_src = torch.empty(m, dtype=torch.int32, device=dev)
        in_eid = torch.empty(m, dtype=torch.int32, device=dev)
        _native.dag_transpose(n, m, out_ptr, out_dst, in_ptr, in_src, in_eid)
        return cls(n, m, root, out_ptr, out_dst, in_ptr, in_src, in_eid, w_cpu, w_gpu, w_xfer,
                   nbytes)

    @classmethod
    def from_taskgraph(cls, graph) -> "DagCSR":
        """A graph without its root node lowers with root = -1 (no node is the
        root): totals, workload ratio and critical path are defined on it as in
        the reference (graph.py:327-332, costs.py:239-253, sim.py:239-247)."""
        return cls.from_host(HostDag.from_taskgraph(graph))

    def validate(self) -> List[str]:
        """``validate`` (graph.py:113-150) on the device, in the reference's message order.

        Covers the checks a CSR can violate (weights, self-loops, cycles,
        kernels without predecessors); the object-model checks (duplicate
        ids/edges, unknown endpoints, root kind) only exist on ``TaskGraph``.
        """
        node_bad = torch.zeros(self.n, dtype=torch.int8, device=self.device)
        edge_bad = torch.zeros(max(self.m, 1), dtype=torch.int8, device=self.device)
        counts, first = _native.validate_dag(self, node_bad, edge_bad)
        ids = self.ids if self.ids is not None else np.arange(self.n, dtype=np.int64)
        out: List[str] = []
        if counts[0] or counts[1]:  # node loop (graph.py:125-129), node order
            nb = node_bad.cpu().numpy()
            for v in np.nonzero(nb & 3)[0]:
                if nb[v] & 1:
                    out.append(f"node {int(ids[v])} has negative weight")
                if nb[v] & 2:
                    out.append(f"SOURCE node {int(ids[v])} must have zero weights")
        if counts[2] or counts[3] or counts[4]:  # edge loop (graph.py:130-140), sorted edges
            eb = edge_bad[:self.m].cpu().numpy()
            bad = np.nonzero(eb)[0]
            src = np.searchsorted(self.out_ptr.cpu().numpy(), bad, side="right") - 1
            dst = self.out_dst.cpu().numpy()[bad]
            for e, u, v in zip(bad, src, dst):
                uu, vv = int(ids[u]), int(ids[v])
                if eb[e] & 1:
                    out.append(f"self-loop on node {uu}")
                if eb[e] & 2:
                    out.append(f"edge ({uu}, {vv}) has negative transfer weight")
                if eb[e] & 4:
                    out.append(f"edge ({uu}, {vv}) has negative byte count")
        if counts[5]:  # topological_order's CycleError (graph.py:171)
            out.append(f"cycle through node {int(ids[first[5]])}")
        if counts[6]:  # graph.py:145-148, node order
            nb = node_bad.cpu().numpy()
            out += [f"initial kernel {int(ids[v])} has no edge from root"
                    for v in np.nonzero(nb & 4)[0]]
        return out

    def struct(self) -> _native.HsDag:
        if self._struct is None:
            p = _native.ptr
            self._struct = _native.HsDag(
                self.n, self.root, self.m, p(self.out_ptr), p(self.out_dst), p(self.in_ptr),
                p(self.in_src), p(self.in_eid), p(self.w_cpu), p(self.w_gpu), p(self.w_xfer),
                p(self.bytes))
        return self._struct

    @property
    def n_kernels(self) -> int:
        return self.n - 1 if self.root >= 0 else self.n

    def kernel_pos(self, idx: np.ndarray) -> np.ndarray:
        if self.root < 0:
            return idx
        return np.where(idx < self.root, idx, idx - 1)

    def twoway(self) -> "TwoWayGraph":
        if self._twoway is None:
            self._twoway = TwoWayGraph.from_host(self.host, self.device)
        return self._twoway


class TwoWayGraph:
    """Undirected kernel graph in the reference's adjacency order (partition.py:153-158).

    Vertex k is the k-th non-root kernel in ascending id order. Neighbour
    lists follow the sorted edge order, each inter-kernel edge (u, v)
    contributing v to u's list and u to v's list. ``edge_*`` is the
    inter-kernel edge list itself in sorted order (what ``_cut_edges`` walks).
    """

    def __init__(self, n, xadj, adjncy, adjwgt, edge_u, edge_v, edge_w):
        self.n = n
        self.xadj, self.adjncy, self.adjwgt = xadj, adjncy, adjwgt
        self.edge_u, self.edge_v, self.edge_w = edge_u, edge_v, edge_w
        self.vwgt = None
        self._struct = None

    @classmethod
    def from_host(cls, h: HostDag, dev) -> "TwoWayGraph":
        n = h.n - 1 if h.root >= 0 else h.n
        keep = (h.src != h.root) & (h.dst != h.root)
        kp = lambda a: (np.where(a < h.root, a, a - 1) if h.root >= 0  # noqa: E731
                        else a).astype(np.int32)
        eu, ev, ew = kp(h.src[keep]), kp(h.dst[keep]), h.w_xfer[keep]
        ne = len(eu)
        node = np.concatenate([eu, ev])
        nbr = np.concatenate([ev, eu])
        pos = np.concatenate([np.arange(ne), np.arange(ne)])
        order = np.lexsort((pos, node))
        t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
        return cls(n, t(_csr_ptr(node, n)), t(nbr[order].astype(np.int32)),
                   t(np.concatenate([ew, ew])[order]), t(eu), t(ev), t(ew))

    def struct(self) -> _native.HsUGraph:
        if self._struct is None:
            p = _native.ptr
            self._struct = _native.HsUGraph(self.n, int(self.adjncy.numel()), p(self.xadj),
                                            p(self.adjncy), p(self.adjwgt), None,
                                            p(self.vwgt) if self.vwgt is not None else None,
                                            None)
        return self._struct


class DagBatch:
    """Many DAGs packed back to back (local indices per graph)."""

    def __init__(self, hosts: Sequence[HostDag], device=None):
        dev = device or _native.device()
        self.device = dev
        self.hosts = list(hosts)
        b = len(hosts)
        self.batch = b
        self.node_counts = np.array([h.n for h in hosts], dtype=np.int64)
        self.edge_counts = np.array([h.m for h in hosts], dtype=np.int64)
        node_off = np.zeros(b + 1, dtype=np.int64)
        edge_off = np.zeros(b + 1, dtype=np.int64)
        np.cumsum(self.node_counts, out=node_off[1:])
        np.cumsum(self.edge_counts, out=edge_off[1:])
        self.node_off_h, self.edge_off_h = node_off, edge_off
        out_ptr, in_ptr, in_src, in_eid = [], [], [], []
        for h in hosts:
            order = h.in_order()
            out_ptr.append(h.out_ptr())
            in_ptr.append(_csr_ptr(h.dst, h.n))
            in_src.append(h.src[order])
            in_eid.append(order)
        cat = lambda xs, dt: torch.from_numpy(  # noqa: E731
            np.ascontiguousarray(np.concatenate(xs) if xs else np.zeros(0, dt), dtype=dt)).to(dev)
        self.node_off = cat([node_off], np.int64)
        self.edge_off = cat([edge_off], np.int64)
        self.root = cat([np.array([h.root for h in hosts], dtype=np.int32)], np.int32)
        self.out_ptr = cat(out_ptr, np.int64)
        self.in_ptr = cat(in_ptr, np.int64)
        self.out_dst = cat([h.dst for h in hosts], np.int32)
        self.in_src = cat(in_src, np.int32)
        self.in_eid = cat(in_eid, np.int32)
        self.w_cpu = cat([h.w_cpu for h in hosts], np.float64)
        self.w_gpu = cat([h.w_gpu for h in hosts], np.float64)
        self.w_xfer = cat([h.w_xfer for h in hosts], np.float64)
        self.bytes = cat([h.bytes for h in hosts], np.int64)
        self._struct = None

    @classmethod
    def from_device(cls, node_counts: np.ndarray, edge_counts: np.ndarray, root, out_ptr,
                    out_dst, in_ptr, in_src, in_eid, w_cpu, w_gpu, w_xfer, nbytes) -> "DagBatch":
        """A batch whose arrays were written on the device (gen.generate_random_dag_batch)."""
        self = cls.__new__(cls)
        self.device = out_ptr.device
        self.hosts = None
        self.batch = len(node_counts)
        self.node_counts = np.asarray(node_counts, dtype=np.int64)
        self.edge_counts = np.asarray(edge_counts, dtype=np.int64)
        self.node_off_h = np.zeros(self.batch + 1, dtype=np.int64)
        self.edge_off_h = np.zeros(self.batch + 1, dtype=np.int64)
        np.cumsum(self.node_counts, out=self.node_off_h[1:])
        np.cumsum(self.edge_counts, out=self.edge_off_h[1:])
        t = lambda a: torch.from_numpy(a).to(self.device)  # noqa: E731
        self.node_off, self.edge_off = t(self.node_off_h), t(self.edge_off_h)
        self.root = root
        self.out_ptr, self.out_dst, self.in_ptr = out_ptr, out_dst, in_ptr
        self.in_src, self.in_eid = in_src, in_eid
        self.w_cpu, self.w_gpu, self.w_xfer, self.bytes = w_cpu, w_gpu, w_xfer, nbytes
        self._struct = None
        return self

    def host_dags(self) -> List[HostDag]:
        """Per-graph HostDag views (numpy) of the batch (ids 0..n_b-1)."""
        if self.hosts is not None:
            return self.hosts
        op = self.out_ptr.cpu().numpy()
        dst = self.out_dst.cpu().numpy()
        wc, wg = self.w_cpu.cpu().numpy(), self.w_gpu.cpu().numpy()
        wx, nb = self.w_xfer.cpu().numpy(), self.bytes.cpu().numpy()
        root = self.root.cpu().numpy()
        out = []
        for b in range(self.batch):
            n0, n1 = self.node_off_h[b], self.node_off_h[b + 1]
            e0, e1 = self.edge_off_h[b], self.edge_off_h[b + 1]
            ptr = op[n0 + b:n1 + b + 1]
            src = np.repeat(np.arange(n1 - n0, dtype=np.int32), np.diff(ptr))
            out.append(HostDag(np.arange(n1 - n0, dtype=np.int64), int(root[b]), src,
                               dst[e0:e1].copy(), wc[n0:n1].copy(), wg[n0:n1].copy(),
                               wx[e0:e1].copy(), nb[e0:e1].copy()))
        self.hosts = out
        return out

    def struct(self) -> _native.HsDagBatch:
        if self._struct is None:
            p = _native.ptr
            self._struct = _native.HsDagBatch(
                self.batch, int(self.node_off_h[-1]), int(self.edge_off_h[-1]),
                p(self.node_off), p(self.edge_off), p(self.root), p(self.out_ptr),
                p(self.out_dst), p(self.in_ptr), p(self.in_src), p(self.in_eid),
                p(self.w_cpu), p(self.w_gpu), p(self.w_xfer), p(self.bytes))
        return self._struct


class TwoWayBatch:
    """Many TwoWayGraphs concatenated (hs_fm2_batch layout)."""

    def __init__(self, hosts: Sequence[HostDag], device=None):
        dev = device or _native.device()
        self.G = len(hosts)
        xadj, adjncy, adjwgt, eu, ev, ew = [], [], [], [], [], []
        node_off, adj_off, edge_off = [0], [0], [0]
        for h in hosts:
            n = h.n - 1
            keep = (h.src != h.root) & (h.dst != h.root)
            kp = lambda a: np.where(a < h.root, a, a - 1).astype(np.int32)  # noqa: E731
            u, v, w = kp(h.src[keep]), kp(h.dst[keep]), h.w_xfer[keep]
            ne = len(u)
            node = np.concatenate([u, v])
            nbr = np.concatenate([v, u])
            pos = np.concatenate([np.arange(ne), np.arange(ne)])
            order = np.lexsort((pos, node))
            xadj.append(_csr_ptr(node, n))
            adjncy.append(nbr[order].astype(np.int32))
            adjwgt.append(np.concatenate([w, w])[order])
            eu.append(u), ev.append(v), ew.append(w)
            node_off.append(node_off[-1] + n)
            adj_off.append(adj_off[-1] + 2 * ne)
            edge_off.append(edge_off[-1] + ne)
        t = lambda xs, dt: torch.from_numpy(  # noqa: E731
            np.ascontiguousarray(np.concatenate(xs) if xs else np.zeros(0, dt), dtype=dt)).to(dev)
        self.node_off_h = np.array(node_off, dtype=np.int64)
        self.node_off = t([self.node_off_h], np.int64)
        self.adj_off = t([np.array(adj_off, dtype=np.int64)], np.int64)
        self.edge_off = t([np.array(edge_off, dtype=np.int64)], np.int64)
        self.xadj = t(xadj, np.int64)
        self.adjncy = t(adjncy, np.int32)
        self.adjwgt = t(adjwgt, np.float64)
        self.edge_u, self.edge_v, self.edge_w = t(eu, np.int32), t(ev, np.int32), t(ew, np.float64)
        self.total_nodes = int(node_off[-1])
        self.max_n = int(max(np.diff(self.node_off_h))) if self.G else 0
