"""CSR-native entry points for graphs beyond the object model (configs 2-4).

* ``layered_dag``      — device generator of the layered fan-in DAG family
                         (100k/1M, 10M/100M) straight into a ``DagCSR``.
* ``integer_weights``  — METIS integerisation of fp64 weights
                         (graphio.py:272-274: ×100, round half up, min 1).
* ``symmetrize``       — K1: DAG -> undirected kernel graph (root dropped).
* ``partition_kway``   — K3-K6 multilevel k-way partitioner.
* ``evaluate_batch``   — K2 integer cut / load / transfer volume for many
                         k-way assignments of one DAG.
* ``levels`` / ``level_order`` / ``critical_path`` — K7 on a ``DagCSR``.

These are additive to the reference API (which stops at 2-way).
"""
from __future__ import annotations

import os
from dataclasses import dataclass
from typing import Dict, Optional, Sequence

import numpy as np
import torch

from . import _native
from .costs import SyntheticCostModel, TransferModel
from .csr import DagCSR


class UGraph:
    """Undirected integer-weighted kernel graph on the device (hs_ugraph_t)."""

    def __init__(self, xadj, adjncy, adjwgt, vwgt, twin=None, unit_weight: int = 1):
        """``adjwgt=None``: every edge weighs ``unit_weight`` (no weight array on
        the device; the partitioner sees unit weights, METIS's adjwgt = NULL)."""
        self.xadj, self.adjncy, self._adjwgt, self.vwgt = xadj, adjncy, adjwgt, vwgt
        self.twin = twin
        self.unit_weight = int(unit_weight)
        self.n = int(vwgt.numel())
        self.nnz = int(adjncy.numel())
        self._struct = None

    @property
    def adjwgt(self) -> torch.Tensor:
        """Per-entry int32 edge weights (materialised when uniform)."""
        if self._adjwgt is None:
            return torch.full((self.nnz,), self.unit_weight, dtype=torch.int32,
                              device=self.adjncy.device)
        return self._adjwgt

    @property
    def weight_scale(self) -> int:
        """Factor between the partitioner's cut and the caller's weights."""
        return self.unit_weight if self._adjwgt is None else 1

    def struct(self):
        if self._struct is None:
            p = _native.ptr
            self._struct = _native.HsUGraph(self.n, self.nnz, p(self.xadj), p(self.adjncy), None,
                                            p(self._adjwgt), None, p(self.vwgt),
                                            p(self.twin) if self.twin is not None else None)
        return self._struct


def _root_out_degree(csr: DagCSR) -> int:
    """Edges leaving the root (one host read per DAG object, then cached)."""
    d = getattr(csr, "_root_outdeg", None)
    if d is None:
        if csr.root < 0:
            raise ValueError("DAG has no root node")
        r = csr.root
        both = torch.stack([csr.out_ptr[r + 1] - csr.out_ptr[r],
                            csr.in_ptr[r + 1] - csr.in_ptr[r]]).tolist()
        if both[1] != 0:  # K1's row layout drops the root's out-list only
            raise ValueError("DAG has edges into the root (validate() it first)")
        d = int(both[0])
        csr._root_outdeg = d
    return d


def _uniform_weight(edge_w_i: torch.Tensor) -> int:
    """The common value of the edge weights if they are all equal and positive, else 0."""
    if edge_w_i.numel() == 0 or os.environ.get("HS_KWAY_WEIGHTS") == "1":
        return 0
    _, lo, hi = _native.int32_stats(edge_w_i)
    return lo if lo == hi and lo > 0 else 0


def layered_dag(n_kernels: int, m_inter: int, seed: int = 0, kind: str = "MA", size: int = 512,
                model=None) -> DagCSR:
    """Layered fan-in DAG generated on the device (see csrc/gen.cu for the family).

    Node weights come from ``model`` (default ``SyntheticCostModel``) for
    (kind, size); every edge carries one size² fp32 matrix (graph.py:195).
    """
    dev = _native.device()
    model = model or SyntheticCostModel()
    n_nodes, m = _native.layered_sizes(n_kernels, m_inter)
    out_ptr = torch.empty(n_nodes + 1, dtype=torch.int64, device=dev)
    in_ptr = torch.empty(n_nodes + 1, dtype=torch.int64, device=dev)
    out_dst = torch.empty(m, dtype=torch.int32, device=dev)
    in_src = torch.empty(m, dtype=torch.int32, device=dev)
    in_eid = torch.empty(m, dtype=torch.int32, device=dev)
    layer_of = torch.empty(n_nodes, dtype=torch.int32, device=dev)
    _native.layered_generate(n_kernels, m_inter, seed, out_ptr, out_dst, in_ptr, in_src, in_eid,
                             layer_of)
    payload = size * size * 4
    nbytes = torch.full((m,), payload, dtype=torch.int64, device=dev)
    w_cpu = w_gpu = w_xfer = None
    csr = DagCSR(n_nodes, m, 0, out_ptr, out_dst, in_ptr, in_src, in_eid, w_cpu, w_gpu, w_xfer,
                 nbytes, ids=None, host=None)
    csr.layer_of = layer_of
    attach_weights_csr(csr, torch.zeros(n_nodes, dtype=torch.int32, device=dev), [kind],
                       torch.full((n_nodes,), size, dtype=torch.int64, device=dev), model)
    return csr


def attach_weights_csr(csr: DagCSR, kind_code: torch.Tensor, kinds: Sequence[str],
                       size: torch.Tensor, model) -> DagCSR:
    """attach_weights (graph.py:308-324) for a device DAG: node v has kind
    ``kinds[kind_code[v]]`` and size ``size[v]`` (device tensors); the root
    gets zero weights; w_cpu / w_gpu / w_xfer are (re)computed on the device
    (hs_attach_weights) from ``model`` and the edges' byte counts. Raises the
    reference's GraphError for the smallest node index without a cost entry
    and the model's CostModelError for a negative byte count."""
    from .costs import _EXACT_SIZE, _closed_form, device_weights
    from .graph import GraphError
    dev = csr.device
    code = kind_code.to(torch.int64)
    closed = _closed_form(model) and int(size.abs().max()) <= min(
        (_EXACT_SIZE.get(k, 0) for k in kinds), default=0) if size.numel() else _closed_form(model)
    if closed:  # one entry per kind, the size per node
        keys = [(k, None) for k in kinds]
        pair = code.to(torch.int32)
    else:  # one entry per distinct (kind, size)
        packed = code << 40 | size.to(torch.int64)
        uniq, inv = torch.unique(packed, return_inverse=True)
        u = uniq.cpu().numpy().tolist()
        keys = [(kinds[x >> 40], x & ((1 << 40) - 1)) for x in u]
        pair = inv.to(torch.int32)
    if 0 <= csr.root < csr.n:
        keys.append(None)
        pair = pair.clone()
        pair[csr.root] = len(keys) - 1
    w_cpu, w_gpu, w_xfer, bad_node, bad_edge = device_weights(
        model, keys, pair.contiguous(), size.to(torch.int64).contiguous(), csr.bytes, device=dev)
    if bad_node >= 0:
        kind, sz = kinds[int(kind_code[bad_node])], int(size[bad_node])
        nid = int(csr.ids[bad_node]) if csr.ids is not None else bad_node
        try:
            model.kernel_time(kind, sz, "CPU")
            model.kernel_time(kind, sz, "GPU")
        except Exception as exc:
            raise GraphError(f"no cost entry for kernel {nid} ({kind}, {sz}): {exc}") from exc
        raise GraphError(f"no cost entry for kernel {nid} ({kind}, {sz})")
    if bad_edge >= 0:
        model.transfer_time(int(csr.bytes[bad_edge]))
    csr.w_cpu, csr.w_gpu, csr.w_xfer = w_cpu, w_gpu, w_xfer
    csr._struct = None
    return csr


def relabeled_dag(csr: DagCSR, seed: int = 0):
    """Input synthesis: the same DAG under a random node numbering (edges and
    weights preserved, out-lists re-sorted). Returns (DagCSR, pi) with
    pi[old node] = new node. The id-order robustness check of the band start."""
    dev = csr.device
    g = torch.Generator(device="cpu").manual_seed(seed)
    pi = torch.randperm(csr.n, generator=g).to(dev)
    src = torch.repeat_interleave(torch.arange(csr.n, device=dev), csr.out_ptr.diff())
    ns, nd = pi[src], pi[csr.out_dst.long()]
    key = ns * csr.n + nd
    key, o = torch.sort(key)
    del key
    out_dst = nd[o].to(torch.int32)
    out_ptr = torch.zeros(csr.n + 1, dtype=torch.int64, device=dev)
    out_ptr[1:] = torch.cumsum(torch.bincount(ns, minlength=csr.n), 0)
    inv = torch.empty_like(pi)
    inv[pi] = torch.arange(csr.n, device=dev)
    new = DagCSR.from_out_csr(int(pi[csr.root].item()), out_ptr, out_dst,
                              csr.w_cpu[inv].contiguous(), csr.w_gpu[inv].contiguous(),
                              csr.w_xfer[o].contiguous(), csr.bytes[o].contiguous())
    return new, pi


def in_order(csr: DagCSR, edge_attr: torch.Tensor) -> torch.Tensor:
    """CSC copy of a per-edge attribute (in-order), for ``symmetrize``."""
    return edge_attr[csr.in_eid.long()].contiguous()


def integer_weights(w: torch.Tensor, scale: int = 100) -> torch.Tensor:
    """``_scaled`` (graphio.py:272-274) elementwise: max(1, floor(w*scale + 0.5)), int32
    (saturated at 2^31 - 1), one device pass (hs_integer_weights)."""
    return _native.integer_weights(w, scale)


def symmetrize(csr: DagCSR, edge_w_i: Optional[torch.Tensor] = None,
               node_w_i: Optional[torch.Tensor] = None,
               edge_w_i_in: Optional[torch.Tensor] = None, unit_ok: bool = True) -> UGraph:
    """K1 on the device; default weights are the integerised w_xfer / w_gpu.

    ``edge_w_i_in`` is the same edge weight in in-order (CSC copy,
    ``edge_w_i[csr.in_eid]``); passing it saves a random gather.
    ``unit_ok``: uniform edge weights produce no weight array (the partitioner
    runs on unit weights and rescales the cut); False always writes them.
    """
    dev = csr.device
    if edge_w_i is None:
        edge_w_i = integer_weights(csr.w_xfer)
    if node_w_i is None:
        node_w_i = integer_weights(csr.w_gpu)
    nk = csr.n - 1
    xadj = torch.empty(nk + 1, dtype=torch.int64, device=dev)
    nnz_cap = 2 * csr.m
    adjncy = torch.empty(nnz_cap, dtype=torch.int32, device=dev)
    vwgt = torch.empty(nk, dtype=torch.int32, device=dev)
    # reverse-entry index for ghost-part refinement: opt-in (its random scatter
    # costs more in K1 than the ghost reads save in K6 on issue-bound passes)
    want_twin = os.environ.get("HS_KWAY_GHOST") == "1" and nnz_cap < 2 ** 31
    twin = torch.empty(nnz_cap, dtype=torch.int32, device=dev) if want_twin else None
    # uniform edge weights (one matrix per transfer): no weight stream at all
    w0 = 0 if want_twin or not unit_ok else _uniform_weight(edge_w_i)
    adjwgt = None if w0 else torch.empty(nnz_cap, dtype=torch.int32, device=dev)
    # entry count = 2 x (edges not leaving the root), cached per DAG: no host
    # read of it after K1
    nnz = 2 * (csr.m - _root_out_degree(csr))
    got = _native.symmetrize(csr, None if w0 else edge_w_i.contiguous(), node_w_i.contiguous(),
                             xadj, adjncy, adjwgt, vwgt,
                             edge_w_i_in.contiguous() if edge_w_i_in is not None and not w0
                             else None, twin, read_nnz=False)
    assert got == -1
    return UGraph(xadj, adjncy[:nnz], adjwgt[:nnz] if adjwgt is not None else None, vwgt,
                  twin[:nnz] if twin is not None else None, unit_weight=w0 or 1)


@dataclass
class KwayResult:
    part: torch.Tensor        # int32 [n] (kernel positions)
    cut: int                  # integer cut, each undirected edge once
    levels: int
    coarsest: int
    max_deviation: float      # max_p |w_p/total - t_p|
    feasible: bool
    refine_passes: int


def partition_kway(graph, k: int, tpwgts: Optional[Sequence[float]] = None, tol: float = 0.03,
                   seed: int = 0, out: Optional[torch.Tensor] = None,
                   reference_start: Optional[bool] = None) -> KwayResult:
    """Multilevel k-way partition (K3-K6) of a ``UGraph`` or ``DagCSR``.

    Balance: |w_p/total - t_p| <= tol for every part (the k-way
    generalisation of partition.py:72); default targets are uniform 1/k.

    ``reference_start`` (default: graphs of at most ``recursive.MAX_KERNELS``
    vertices) adds the reference heuristic applied recursively
    (``recursive.py``) as a start partition; the partitioner refines it with
    its own candidates and returns the best, so the cut never exceeds that
    baseline's when the baseline meets the balance constraint.
    """
    from . import recursive
    if not isinstance(graph, UGraph):
        return partition_dag(graph, k, tpwgts, tol, seed, out=out,
                             reference_start=reference_start)
    ug = graph
    if tpwgts is None:
        tpwgts = [1.0 / k] * k
    if len(tpwgts) != k:
        raise ValueError("need one target fraction per part")
    part = out if out is not None else torch.empty(ug.n, dtype=torch.int32, device=ug.xadj.device)
    if reference_start is None:
        reference_start = 2 <= k and 2 <= ug.n <= recursive.MAX_KERNELS
    starts = recursive.reference_recursive_start(ug, k, tpwgts, tol) if reference_start else None
    st = _native.partition_kway(ug, k, tpwgts, tol, seed, part, starts)
    return KwayResult(part, st[0] * ug.weight_scale, st[1], st[2], st[3] / 1e9, bool(st[4]),
                      st[5])


def permute_ugraph(ug: UGraph, perm: torch.Tensor, inv: torch.Tensor) -> UGraph:
    """``ug`` relabelled: vertex i of the result is vertex perm[i] (hs_ugraph_permute)."""
    xadj, adjncy, adjwgt, vwgt = _native.ugraph_permute(ug, perm, inv)
    return UGraph(xadj, adjncy, adjwgt, vwgt, unit_weight=ug.unit_weight)


def band_order(csr: DagCSR, order: str = "auto"):
    """The vertex order the band start cuts: None (kernel positions) or the
    (perm, inv) of the longest-path level order.

    ``order``: "ids" keeps positions; "levels" always relabels; "auto"
    relabels only DAGs not numbered in topological order (one read per row,
    ``hs_dag_is_topological``): creation-order numbering (the reference's
    generator, graph.py:180-305; the tiled-Cholesky DAG) already follows the
    layers, an arbitrary numbering does not.
    """
    if order not in ("auto", "ids", "levels"):
        raise ValueError("order must be 'auto', 'ids' or 'levels'")
    if order == "auto":
        topo = getattr(csr, "_topological", None)
        if topo is None:
            topo = csr._topological = _native.dag_is_topological(csr)
        if topo:
            return None
    if order == "ids":
        return None
    lv, _, _, nl = _native.levels(csr, 0)
    return _native.level_permutation(csr, lv, nl)


def partition_dag(csr: DagCSR, k: int, tpwgts: Optional[Sequence[float]] = None,
                  tol: float = 0.03, seed: int = 0, edge_w_i: Optional[torch.Tensor] = None,
                  node_w_i: Optional[torch.Tensor] = None,
                  edge_w_i_in: Optional[torch.Tensor] = None, order: str = "auto",
                  out: Optional[torch.Tensor] = None,
                  reference_start: Optional[bool] = None) -> KwayResult:
    """K1 + K3-K6 on a task DAG, the band start cut in ``band_order(csr, order)``.

    The result's ``part`` is indexed by kernel position whatever the order.
    """
    ug = symmetrize(csr, edge_w_i, node_w_i, edge_w_i_in)
    po = band_order(csr, order)
    if po is None:
        return partition_kway(ug, k, tpwgts, tol, seed, out=out, reference_start=reference_start)
    perm, inv = po
    r = partition_kway(permute_ugraph(ug, perm, inv), k, tpwgts, tol, seed,
                       reference_start=reference_start)
    part = out if out is not None else torch.empty_like(r.part)
    r.part = _native.parts_unpermute(perm, r.part, part)
    return r


def evaluate_batch(csr: DagCSR, parts: torch.Tensor, k: int,
                   node_w_i: Optional[torch.Tensor] = None,
                   check: bool = True) -> Dict[str, torch.Tensor]:
    """K2 for B k-way assignments (int32 [B, n], node index space incl. root).

    A part id outside [0, k) on a non-root node is never used as an index: the
    kernel flags that assignment (cut_edges = xfer_count = -1). ``check``
    (default) turns a flagged assignment into ValueError (one host read);
    ``check=False`` leaves the flag to the caller and keeps the call async.
    """
    if node_w_i is None:
        node_w_i = integer_weights(csr.w_gpu).to(torch.int64)
    if parts.dim() == 1:
        parts = parts.unsqueeze(0)
    out = _native.evaluate_kway(csr, parts.contiguous(), k, node_w_i.contiguous())
    if check:
        bad = torch.nonzero(out["cut_edges"] < 0).flatten().tolist()
        if bad:
            raise ValueError(f"assignment {bad[0]} has a part id outside [0, {k})")
    return out


def kernel_to_node_parts(csr: DagCSR, kpart: torch.Tensor) -> torch.Tensor:
    """Kernel-position part array -> node-index part array (root gets part 0)."""
    r = csr.root
    return torch.cat([kpart[:r], kpart.new_zeros(1), kpart[r:]]).contiguous()


def levels(csr: DagCSR, mode: int = 0):
    """Longest-path level per node and the critical path (K7)."""
    return _native.levels(csr, mode)


def assigned_makespan(csr: DagCSR, part: torch.Tensor, gpu_parts: Optional[Sequence[int]] = None,
                      k: Optional[int] = None):
    """Level-synchronous makespan of a k-way assignment (node index space, K7 mode 3).

    Parts listed in ``gpu_parts`` run at GPU speed (w_gpu), the others at CPU
    speed; default: every part is a GPU. Cross-part edges add their transfer
    time; the root's outputs start in host memory. Returns (makespan, finish).
    """
    k = int(k if k is not None else int(part.max().item()) + 1)
    dev = torch.zeros(k, dtype=torch.int8, device=csr.device)
    if gpu_parts is None:
        dev.fill_(1)
    else:
        dev[list(gpu_parts)] = 1
    return _native.assigned_makespan(csr, part.to(torch.int32).contiguous(), dev)


def level_order(csr: DagCSR) -> torch.Tensor:
    lv, _, _, nl = _native.levels(csr, 0)
    return _native.level_order(csr, lv, nl)


# ---------------------------------------------------------------------------
# Sharded partition (config 4 at 2/4/8 GPUs): rank r owns a contiguous range
# of kernel positions; see csrc/dist.cuh for the exchange protocol.
# ---------------------------------------------------------------------------

def undirected_degrees(csr: DagCSR) -> torch.Tensor:
    """Degree of every kernel in the symmetrised graph (root edges dropped), int64."""
    deg = (csr.in_ptr[1:] - csr.in_ptr[:-1]) + (csr.out_ptr[1:] - csr.out_ptr[:-1])
    r = csr.root
    fed = csr.out_dst[int(csr.out_ptr[r]):int(csr.out_ptr[r + 1])].long()
    deg = deg.clone()
    deg[fed] -= 1
    return torch.cat([deg[:r], deg[r + 1:]])


def split_bounds(deg_cumsum: np.ndarray, nranks: int) -> list:
    """Rank boundaries over kernel positions balancing adjacency entries.

    deg_cumsum[i] = entries of kernels 0..i (inclusive). Boundary b_r (r = 1..P-1)
    is the first position whose inclusive sum exceeds r/P of the total; every
    rank gets at least one kernel. Pure integer function: every rank derives
    the same ranges.
    """
    n = int(len(deg_cumsum))
    if nranks < 1 or nranks > n:
        raise ValueError(f"need 1 <= ranks <= {n} kernels (got {nranks})")
    total = int(deg_cumsum[-1]) if n else 0
    b = [0]
    for r in range(1, nranks):
        t = (total * r) // nranks
        x = int(np.searchsorted(deg_cumsum, t, side="right"))
        x = max(x, b[-1] + 1)
        x = min(x, n - (nranks - r))
        b.append(x)
    b.append(n)
    return [(b[i], b[i + 1]) for i in range(nranks)]


def shard_ranges(csr: DagCSR, nranks: int) -> list:
    cs = torch.cumsum(undirected_degrees(csr), 0).cpu().numpy()
    return split_bounds(cs, nranks)


def symmetrize_range(csr: DagCSR, kv0: int, kv1: int, edge_w_i: Optional[torch.Tensor] = None,
                     node_w_i: Optional[torch.Tensor] = None,
                     edge_w_i_in: Optional[torch.Tensor] = None,
                     cap: Optional[int] = None) -> UGraph:
    """K1 for the rows of kernel positions [kv0, kv1) (global neighbour ids).

    ``cap`` = the rows' adjacency entries when known (saves a host round trip).
    """
    dev = csr.device
    if edge_w_i is None:
        edge_w_i = integer_weights(csr.w_xfer)
    if node_w_i is None:
        node_w_i = integer_weights(csr.w_gpu)
    nl = kv1 - kv0
    if cap is None:
        cap = int(undirected_degrees(csr)[kv0:kv1].sum().item()) if nl else 0
    xadj = torch.empty(nl + 1, dtype=torch.int64, device=dev)
    adjncy = torch.empty(max(cap, 1), dtype=torch.int32, device=dev)
    # the uniformity test reads the whole weight array: every rank decides alike
    w0 = _uniform_weight(edge_w_i)
    adjwgt = None if w0 else torch.empty(max(cap, 1), dtype=torch.int32, device=dev)
    vwgt = torch.empty(max(nl, 1), dtype=torch.int32, device=dev)
    nnz = _native.symmetrize_range(csr, kv0, kv1, None if w0 else edge_w_i.contiguous(),
                                   node_w_i.contiguous(), xadj, adjncy, adjwgt, vwgt,
                                   edge_w_i_in.contiguous() if edge_w_i_in is not None and not w0
                                   else None)
    assert nnz == cap
    return UGraph(xadj, adjncy[:nnz], adjwgt[:nnz] if adjwgt is not None else None, vwgt[:nl],
                  unit_weight=w0 or 1)


# ---- row-range input for one rank (e2e at N > 1) -------------
# Rank r of a sharded partition needs, for its kernel rows [kv0, kv1), only
# their in- and out-lists (global neighbour ids), the out- and in-order edge
# weights of those lists, their node weights, and — the halo K1's row starts
# need — which of its rows the root feeds. row_slice packs exactly that, on
# the caller's side, as a small DAG: node 0 stands in for the root (no inputs,
# one edge to every local row the root feeds, local ids), nodes 1..nl are the
# rows. K1 (hs_symmetrize_range over all local rows) then writes the same
# rows, entry for entry, as over the whole graph.
ROW_SLICE_KEYS = ("out_ptr", "out_dst", "in_ptr", "in_src", "ew", "ew_in", "nw")


def row_slice(out_ptr, out_dst, in_ptr, in_src, ew, ew_in, nw, kv0: int, kv1: int) -> dict:
    """numpy (caller-side) slice of a DAG whose root is node 0 for kernel rows
    [kv0, kv1): a dict of the local DAG's arrays (ROW_SLICE_KEYS) plus
    ``nnz`` (undirected entries of the rows), ``kv0``, ``kv1``."""
    v0, v1 = kv0 + 1, kv1 + 1  # node ids of the rows (root = node 0)
    o0, o1 = int(out_ptr[v0]), int(out_ptr[v1])
    i0, i1 = int(in_ptr[v0]), int(in_ptr[v1])
    starts = in_ptr[v0:v1]
    nonempty = in_ptr[v0 + 1:v1 + 1] > starts
    fed = np.zeros(v1 - v0, dtype=bool)
    fed[nonempty] = in_src[starts[nonempty]] == 0  # in-lists ascend: the root sorts first
    fed_ids = (np.nonzero(fed)[0] + 1).astype(np.int32)
    R = len(fed_ids)
    l_out_ptr = np.empty(v1 - v0 + 2, dtype=np.int64)
    l_out_ptr[0] = 0
    l_out_ptr[1:] = R + (out_ptr[v0:v1 + 1] - o0)
    l_in_ptr = np.empty(v1 - v0 + 2, dtype=np.int64)
    l_in_ptr[0] = 0
    l_in_ptr[1:] = in_ptr[v0:v1 + 1] - i0
    return {"out_ptr": l_out_ptr,
            "out_dst": np.concatenate([fed_ids, out_dst[o0:o1].astype(np.int32)]),
            "in_ptr": l_in_ptr, "in_src": np.ascontiguousarray(in_src[i0:i1], dtype=np.int32),
            "ew": np.concatenate([np.zeros(R, np.int32), ew[o0:o1].astype(np.int32)]),
            "ew_in": np.ascontiguousarray(ew_in[i0:i1], dtype=np.int32),
            "nw": np.concatenate([np.zeros(1, np.int32), nw[v0:v1].astype(np.int32)]),
            "nnz": (i1 - i0) - R + (o1 - o0), "kv0": kv0, "kv1": kv1}


def symmetrize_slice(sl: dict, unit_weight: Optional[int] = None) -> UGraph:
    """K1 of one rank's rows from its row_slice (arrays as device tensors):
    the UGraph symmetrize_range(csr, kv0, kv1, ...) builds from the whole DAG.
    ``unit_weight``: the sharded graph's common edge weight (0 if weights
    differ) — every rank must decide alike, so a caller holding only a slice
    passes the decision over all ranks' weights; None decides on this slice."""
    t = {k: sl[k] for k in ROW_SLICE_KEYS}
    n_loc = int(t["out_ptr"].numel()) - 1
    nl = n_loc - 1
    dev = t["out_ptr"].device
    if unit_weight is None:
        R = int(t["out_ptr"][1].item())
        both = torch.cat([t["ew"][R:], t["ew_in"]])
        unit_weight = _uniform_weight(both)
    g = DagCSR(n_loc, int(t["out_dst"].numel()), 0, t["out_ptr"], t["out_dst"], t["in_ptr"],
               t["in_src"], None, None, None, None, None)
    cap = int(sl["nnz"])
    xadj = torch.empty(nl + 1, dtype=torch.int64, device=dev)
    adjncy = torch.empty(max(cap, 1), dtype=torch.int32, device=dev)
    adjwgt = None if unit_weight else torch.empty(max(cap, 1), dtype=torch.int32, device=dev)
    vwgt = torch.empty(max(nl, 1), dtype=torch.int32, device=dev)
    nnz = _native.symmetrize_range(g, 0, nl, None if unit_weight else t["ew"], t["nw"], xadj,
                                   adjncy, adjwgt, vwgt, None if unit_weight else t["ew_in"])
    assert nnz == cap
    return UGraph(xadj, adjncy[:nnz], adjwgt[:nnz] if adjwgt is not None else None, vwgt[:nl],
                  unit_weight=unit_weight or 1)


class PartitionGroup:
    """Exchange arenas of a sharded partition, one whole device allocation per rank.

    mode "loopback": every rank's arena on this GPU (ranks run as host threads on
    separate streams) — the exact cross-rank protocol on one device.
    mode "ipc": this process is rank `rank` of a torch.distributed group with one
    process per GPU; peers' arenas are CUDA-IPC mappings.
    """

    def __init__(self, n_global: int, nranks: int, mode: str = "loopback", rank: int = 0,
                 group=None):
        from .cholesky import _Buf, _ipc_handle, _ipc_open
        if not 1 <= nranks <= 8:
            raise ValueError("1..8 ranks")
        self.n_global, self.nranks, self.mode = n_global, nranks, mode
        self.bytes = _native.kway_dist_arena_bytes(n_global)
        if mode == "loopback":
            self.bufs = [_Buf(self.bytes) for _ in range(nranks)]
            for b in self.bufs:
                b.fill_bytes(0)
            self.ptrs = [b.data_ptr() for b in self.bufs]
        elif mode == "ipc":
            import torch.distributed as dist
            import ctypes
            me = _Buf(self.bytes)
            me.fill_bytes(0)
            torch.cuda.synchronize()
            self.bufs = [me]
            h = ctypes.create_string_buffer(64)
            _native.check(_ipc_handle(me.data_ptr(), h))
            allh = [None] * nranks
            dist.all_gather_object(allh, h.raw, group=group)
            self.ptrs = []
            for q in range(nranks):
                if q == rank:
                    self.ptrs.append(me.data_ptr())
                    continue
                p = ctypes.c_void_p()
                _native.check(_ipc_open(allh[q], ctypes.byref(p)))
                self.ptrs.append(p.value)
            dist.barrier(group=group)  # every arena zeroed before any rank's first flag
        else:
            raise ValueError(mode)
        torch.cuda.synchronize()

    def dist(self, rank: int):
        d = _native.HsDist()
        d.rank, d.size, d.arena_bytes = rank, self.nranks, self.bytes
        d.mode = 1 if self.mode == "loopback" else 0
        for q, p in enumerate(self.ptrs):
            d.arena[q] = p
        return d


def partition_kway_shard(ug_local: UGraph, v0: int, n_global: int, group: PartitionGroup,
                         rank: int, k: int, tpwgts: Optional[Sequence[float]] = None,
                         tol: float = 0.03, seed: int = 0,
                         out: Optional[torch.Tensor] = None) -> KwayResult:
    """One rank's share of a sharded partition; returns the WHOLE partition (every rank)."""
    if tpwgts is None:
        tpwgts = [1.0 / k] * k
    if len(tpwgts) != k:
        raise ValueError("need one target fraction per part")
    part = out if out is not None else torch.empty(n_global, dtype=torch.int32,
                                                   device=ug_local.xadj.device)
    st = _native.partition_kway_dist(ug_local, v0, n_global, group.dist(rank), k, tpwgts, tol,
                                     seed, part)
    return KwayResult(part, st[0] * ug_local.weight_scale, st[1], st[2], st[3] / 1e9,
                      bool(st[4]), st[5])


def partition_kway_loopback(csr: DagCSR, nranks: int, k: int,
                            tpwgts: Optional[Sequence[float]] = None, tol: float = 0.03,
                            seed: int = 0, group: Optional[PartitionGroup] = None,
                            shards: Optional[list] = None):
    """All ranks of a sharded partition on this GPU (one host thread + stream per rank).

    Returns the list of per-rank KwayResults (each holds the whole partition).
    """
    import threading
    n_global = csr.n - 1
    ranges = shard_ranges(csr, nranks)
    if shards is None:
        ew = integer_weights(csr.w_xfer)
        shards = [symmetrize_range(csr, a, b, ew, integer_weights(csr.w_gpu), in_order(csr, ew))
                  for a, b in ranges]
    group = group or PartitionGroup(n_global, nranks)
    dev = csr.device
    cur = torch.cuda.current_stream()
    streams = [torch.cuda.Stream(device=dev) for _ in range(nranks)]
    for st in streams:
        st.wait_stream(cur)
    out, err = [None] * nranks, [None] * nranks

    def run(r):
        try:
            torch.cuda.set_device(dev)
            with torch.cuda.stream(streams[r]):
                out[r] = partition_kway_shard(shards[r], ranges[r][0], n_global, group, r, k,
                                              tpwgts, tol, seed)
        except BaseException as e:  # noqa: BLE001 — re-raised on the caller's thread
            err[r] = e

    th = [threading.Thread(target=run, args=(r,)) for r in range(nranks)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for st in streams:
        cur.wait_stream(st)
    for e in err:
        if e is not None:
            raise e
    return out
