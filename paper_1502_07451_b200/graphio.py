"""DOT ingestion and the METIS wire boundary (row 3) on the device.

* ``parse_dot(text) -> TaskGraph`` (graphio.py:79-199): ``hs_dot_parse``
  tokenises the text in HBM, one thread per line, with the reference's DOT
  subset (header, comments, statement split, edge / node / attribute grammar,
  closing brace), deduplicates node names in a device hash table, assigns ids
  as graphio.py:145-158 does and converts every numeric attribute with a
  device restatement of CPython's ``float()`` (Eisel-Lemire). The host turns
  the arrays into ``KernelNode``/``DataEdge`` objects (the return type) and
  formats ``DotParseError`` messages from the byte spans the device reports.
  ``parse_dot_csr(text) -> DagCSR`` keeps the whole graph on the device.

Same names, arguments and errors as the reference's graphio
(pkg/src/hetsched/graphio.py:272-339):

* ``emit_metis(graph, node_weight_source, scale) -> str``: the undirected
  METIS graph of the kernels (graphio.py:277-304). Integerisation
  ``max(1, floor(w*scale + 0.5))`` (graphio.py:272-274) on the device, K1
  symmetrisation, then ``hs_emit_metis`` formats every line in HBM (row byte
  lengths, a scan, one warp per row writing digits).
* ``parse_partition_file(text, graph, targets, node_weight_source, tolerance)
  -> Partition`` (graphio.py:307-330): ``hs_parse_partition`` splits lines
  like ``str.splitlines``, strips ASCII whitespace and decides every line that
  is a plain signed decimal. The few lines it cannot decide (non-ASCII
  whitespace, ``1_0``-style digit separators, more than 18 digits) come back
  with their line numbers and are finished with Python's own ``int()`` so that
  values and error messages match the reference exactly.
* ``emit_partition_file(partition, graph) -> str`` (graphio.py:333-339).

``emit_metis_csr`` / ``parse_partition_bytes`` are the CSR-native forms for
graphs beyond the object model (config 4: 10M vertices, ~2.6 GB of text).
"""
from __future__ import annotations

import ctypes
import re
from typing import Dict, List, Optional, Tuple

import numpy as np
import torch

from . import _native
from .costs import PartitionTargets
from .csr import DagCSR
from .graph import CPU, GPU, SOURCE_KIND, DataEdge, KernelNode, TaskGraph
from .partition import Partition, PartitionError, _finish

_P = ctypes.c_void_p
_emit = _native._opt("hs_emit_metis", _P, _P, ctypes.c_int64, _P, _P)
_parse = _native._opt("hs_parse_partition", _P, ctypes.c_int64, ctypes.c_int32, _P, _P, _P,
                      ctypes.c_int32, _P, _P)


# ---- canonical DOT emission (graphio.py:27-47, 221-270) ---------------------
# Text formatting of the object model: the trace products annotated_dot /
# emit_partitioned_dot are built on it.
_ID_RE = re.compile(r"[A-Za-z_][A-Za-z0-9_]*$")
_NUM_RE = re.compile(r"-?(\.\d+|\d+(\.\d*)?)$")
CPU_COLOR = "lightblue"
GPU_COLOR = "palegreen"


def _quote(value: str) -> str:
    """graphio.py:32-35"""
    if _ID_RE.match(value) or _NUM_RE.match(value):
        return value
    return '"' + value.replace('"', '\\"') + '"'


def _fmt_attrs(pairs: List[Tuple[str, str]]) -> str:
    return "[" + ", ".join(f"{k}={_quote(v)}" for k, v in pairs) + "]"


def _node_attr_pairs(n) -> List[Tuple[str, str]]:
    """graphio.py:221-225 (floats as repr)"""
    return [("kind", n.kind), ("size", str(n.size)), ("weight_cpu", repr(n.weight_cpu)),
            ("weight_gpu", repr(n.weight_gpu))] + list(getattr(n, "attrs", ()))


def _edge_attr_pairs(e) -> List[Tuple[str, str]]:
    """graphio.py:228-231"""
    return [("bytes", str(e.bytes)), ("weight_xfer", repr(e.weight_xfer))] + \
        list(getattr(e, "attrs", ()))


def emit_dot(graph: TaskGraph,
             node_extra: Optional[Dict[int, List[Tuple[str, str]]]] = None,
             edge_extra: Optional[Dict[Tuple[int, int], List[Tuple[str, str]]]] = None) -> str:
    """Canonical DOT: nodes ascending by id, then edges by (src, dst) (graphio.py:234-250)."""
    node_extra = node_extra or {}
    edge_extra = edge_extra or {}
    lines = [f"digraph {graph.name} {{"]
    for nid in sorted(graph.nodes):
        pairs = _node_attr_pairs(graph.nodes[nid]) + node_extra.get(nid, [])
        lines.append(f"  n{nid} {_fmt_attrs(pairs)};")
    for (u, v) in sorted(graph.edges):
        pairs = _edge_attr_pairs(graph.edges[(u, v)]) + edge_extra.get((u, v), [])
        lines.append(f"  n{u} -> n{v} {_fmt_attrs(pairs)};")
    lines.append("}")
    return "\n".join(lines) + "\n"


def emit_partitioned_dot(graph: TaskGraph, partition: Partition) -> str:
    """emit_dot with part / fill colour per group and dashed red cut edges (graphio.py:253-270)."""
    for nid in graph.kernel_ids():
        if nid not in partition.assignment:
            raise PartitionError(f"partition is missing kernel {nid}")
    node_extra: Dict[int, List[Tuple[str, str]]] = {}
    for nid, group in partition.assignment.items():
        color = CPU_COLOR if group == CPU else GPU_COLOR
        node_extra[nid] = [("part", group), ("style", "filled"), ("fillcolor", color)]
    node_extra[graph.root] = [("part", CPU), ("style", "filled"), ("fillcolor", CPU_COLOR)]
    edge_extra: Dict[Tuple[int, int], List[Tuple[str, str]]] = {}
    for (u, v) in sorted(graph.edges):
        if u == graph.root or v == graph.root:
            continue
        if partition.assignment[u] != partition.assignment[v]:
            edge_extra[(u, v)] = [("style", "dashed"), ("color", "red")]
    return emit_dot(graph, node_extra, edge_extra)


# ---- DOT parsing (graphio.py:20-25, 79-199) -----------------------------------
KNOWN_NODE_ATTRS = ("kind", "size", "weight_cpu", "weight_gpu")
KNOWN_EDGE_ATTRS = ("bytes", "weight_xfer")
STYLE_ATTRS = ("part", "color", "style", "fillcolor", "device", "start", "end")
# attribute classes of hs_dot_parse
_K_KIND, _K_SIZE, _K_WCPU, _K_WGPU, _K_BYTES, _K_WXFER, _K_STYLE, _K_OTHER = range(8)
_NODE_EXTRA = np.array([0, 0, 0, 0, 1, 1, 0, 1], dtype=bool)  # not known, not style
_EDGE_EXTRA = np.array([1, 1, 1, 1, 0, 0, 0, 1], dtype=bool)


class DotParseError(Exception):
    """graphio.py:20-25"""

    def __init__(self, message: str, line: int, column: int = 1):
        super().__init__(f"line {line}, column {column}: {message}")
        self.line = line
        self.column = column


def _unquote(raw: str) -> str:
    """_unquote_name / attribute value unquoting (graphio.py:57-58, 73-76)."""
    return raw[1:-1].replace('\\"', '"') if raw.startswith('"') else raw


class _DotText:
    def __init__(self, data: bytes):
        self.data = data

    def raw(self, a: int, b: int) -> str:
        return self.data[a:b].decode("utf-8", "surrogatepass")

    def value(self, a: int, b: int) -> str:
        return _unquote(self.raw(a, b))


def _dot_error(t: _DotText, info) -> DotParseError:
    st, line = info.status, info.err_line
    if st == 1:
        return DotParseError(f"expected a digraph header, got {t.raw(info.err_a, info.err_b)!r}",
                             line)
    if st == 2:
        return DotParseError("undirected graphs are not supported", line)
    if st == 3:
        return DotParseError(f"cannot parse statement {t.raw(info.err_a, info.err_b)!r}", line)
    if st == 4:
        text = t.raw(info.err_a, info.err_b)
        pos = len(t.raw(info.err_a, info.err_c))
        return DotParseError(f"bad attribute syntax near {text[pos:pos + 20]!r}", line, pos + 1)
    if st == 5:
        return DotParseError("no digraph found", line)
    return DotParseError("missing closing brace", line)


def _dot_device(text: str):
    """hs_dot_parse + the reference's error for a rejected text."""
    data = text.encode("utf-8", "surrogatepass")
    info, handle = _native.dot_parse(data)
    t = _DotText(data)
    if info.status:
        raise _dot_error(t, info)
    return t, info, handle


def _dot_values(t: _DotText, info, a: dict) -> List[Tuple[int, object]]:
    """Values the device left to CPython (int(float()) beyond int64) and the
    first conversion failure, in the reference's evaluation order (graphio.py:160-183): the
    failing literal is re-evaluated here so the exception is Python's own."""
    U = info.n_names
    fail = info.conv_err >> 3 if info.conv_err >= 0 else None
    fixes = []
    for order, attr in a["slow"].reshape(-1, 2):
        order, attr = int(order), int(attr)
        val = t.value(int(a["v0"][attr]), int(a["v1"][attr]))
        is_int = (order < 3 * U and order % 3 == 0) or (order >= 3 * U and (order - 3 * U) % 2 == 0)
        try:
            x = int(float(val)) if is_int else float(val)
        except (ValueError, OverflowError):
            if fail is None or order < fail:
                fail = order
            continue
        fixes.append((order, x))
    if fail is not None:
        # the literal behind `fail` raises the reference's exception
        if fail < 3 * U:
            r, f = divmod(fail, 3)
            owner_ok = a["owner"] == r
            key = (_K_SIZE, _K_WCPU, _K_WGPU)[f]
        else:
            e, f = divmod(fail - 3 * U, 2)
            owner_ok = a["owner"] == -1 - e
            key = (_K_BYTES, _K_WXFER)[f]
        idx = np.nonzero(owner_ok & (a["cls"] == key))[0][-1]
        val = t.value(int(a["v0"][idx]), int(a["v1"][idx]))
        if key in (_K_SIZE, _K_BYTES):
            int(float(val))
        else:
            float(val)
        raise ValueError(f"could not convert string to float: {val!r}")  # not reached
    return fixes


def _extras(t: _DotText, a: dict, node: bool) -> Dict[int, Tuple[Tuple[str, str], ...]]:
    owner, cls = a["owner"], a["cls"]
    sel = (owner >= 0) & _NODE_EXTRA[cls] if node else (owner < 0) & _EDGE_EXTRA[cls]
    idx = np.nonzero(sel)[0]
    out: Dict[int, List[Tuple[str, str]]] = {}
    for i in idx[np.argsort(owner[idx] if node else -1 - owner[idx], kind="stable")]:
        o = int(owner[i]) if node else -1 - int(owner[i])
        out.setdefault(o, []).append((t.raw(int(a["k0"][i]), int(a["k1"][i])),
                                      t.value(int(a["v0"][i]), int(a["v1"][i]))))
    return {k: tuple(v) for k, v in out.items()}


def parse_dot(text: str) -> TaskGraph:
    """Parse the supported DOT subset into a TaskGraph (graphio.py:79-199).

    Node names of the form ``n<int>`` (or bare integers) keep that id; other
    names get sequential ids in order of appearance. A zero-weight root is
    synthesized and wired to all in-degree-0 kernels if no SOURCE node is
    declared. Tokenising, name resolution and numeric conversion run on the
    device (``hs_dot_parse``).
    """
    t, info, h = _dot_device(text)
    try:
        a = h.fetch()
    finally:
        h.close()
    fixes = _dot_values(t, info, a)
    U, E = info.n_names, info.n_edges
    name = "task"
    if info.name_b >= 0:
        name = _unquote(t.raw(info.name_b, info.name_e))
    ids = a["id"].tolist()
    # kind strings: one decode per distinct value
    kinds = ["K"] * U
    ka = a["kind_attr"]
    has = np.nonzero(ka >= 0)[0]
    if has.size:
        uh, first, inv = np.unique(a["kind_hash"][has], return_index=True, return_inverse=True)
        names = [t.value(int(a["v0"][ka[has[j]]]), int(a["v1"][ka[has[j]]])) for j in first]
        for j, r in enumerate(has.tolist()):
            kinds[r] = names[inv[j]]
    nx = _extras(t, a, True)
    ex = _extras(t, a, False)
    size, wc, wg = a["size"].tolist(), a["w_cpu"].tolist(), a["w_gpu"].tolist()
    nb, wx = a["bytes"].tolist(), a["w_xfer"].tolist()
    for order, x in fixes:  # literals finished by CPython
        if order < 3 * U:
            r, f = divmod(order, 3)
            (size, wc, wg)[f][r] = x
        else:
            e, f = divmod(order - 3 * U, 2)
            (nb, wx)[f][e] = x
    nodes = [KernelNode(id=ids[r], kind=kinds[r], size=size[r], weight_cpu=wc[r],
                        weight_gpu=wg[r], attrs=nx.get(r, ())) for r in range(U)]
    src, dst = a["src"].tolist(), a["dst"].tolist()
    edges = [DataEdge(src=ids[src[e]], dst=ids[dst[e]], bytes=nb[e], weight_xfer=wx[e],
                      attrs=ex.get(e, ())) for e in range(E)]
    if info.root_rank >= 0:
        root_id = ids[info.root_rank]
    else:
        root_id = 0 if 0 not in set(ids) else int(info.max_id) + 1
        no_pred = np.nonzero(a["has_pred"] == 0)[0]
        order = no_pred[np.argsort(a["id"][no_pred], kind="stable")]
        nodes.insert(0, KernelNode(root_id, SOURCE_KIND, 0))
        edges.extend(DataEdge(root_id, ids[r]) for r in order.tolist())
    return TaskGraph(nodes, edges, root=root_id, name=name)


def parse_dot_csr(text, device=None) -> DagCSR:
    """The graph ``parse_dot(text)`` would return, as a device CSR built on the
    device (``hs_dot_csr``): node ids ascending (``.ids``), edges by (src, dst)
    with a later duplicate winning, the synthesized root and its edges. For
    texts whose node count makes the object model impractical (config 2/4).
    Byte counts beyond int64 (Python ints) have no CSR form."""
    data = text if isinstance(text, (bytes, bytearray)) else text.encode("utf-8", "surrogatepass")
    info, h = _native.dot_parse(bytes(data), device)
    t = _DotText(bytes(data))
    if info.status:
        raise _dot_error(t, info)
    fixes, a = [], None
    try:
        if info.conv_err >= 0 or info.n_slow:
            a = h.fetch()
            fixes = _dot_values(t, info, a)  # raises the first conversion error
        root, out_ptr, out_dst, ids, w_cpu, w_gpu, w_xfer, nbytes = h.csr()
    finally:
        h.close()
    ids_h = ids.cpu().numpy()
    U = info.n_names
    for order, x in fixes:
        if order < 3 * U:
            r, f = divmod(order, 3)
            if f:  # size is not part of the CSR
                (w_cpu, w_gpu)[f - 1][int(np.searchsorted(ids_h, a["id"][r]))] = x
            continue
        e, f = divmod(order - 3 * U, 2)
        if f == 0:
            raise _native.NativeError(-3, "parse_dot_csr: bytes beyond int64 have no CSR form: "
                                      "use parse_dot")
        su, sv = a["id"][a["src"][e]], a["id"][a["dst"][e]]
        same = np.nonzero((a["id"][a["src"]] == su) & (a["id"][a["dst"]] == sv))[0]
        if same[-1] != e:  # a later declaration of the same edge wins
            continue
        i, j = int(np.searchsorted(ids_h, su)), int(np.searchsorted(ids_h, sv))
        lo, hi = int(out_ptr[i]), int(out_ptr[i + 1])
        row = out_dst[lo:hi].cpu().numpy()
        w_xfer[lo + int(np.searchsorted(row, j))] = x
    csr = DagCSR.from_out_csr(root, out_ptr, out_dst, w_cpu, w_gpu, w_xfer, nbytes)
    csr.ids = ids_h
    return csr


def _scaled(w: torch.Tensor, scale: int) -> torch.Tensor:
    """graphio.py:272-274 elementwise: max(1, floor(w*scale + 0.5)) as int32."""
    return torch.clamp(torch.floor(w * scale + 0.5), min=1).to(torch.int32)


def emit_metis_csr(csr: DagCSR, node_weight_source: str = GPU, scale: int = 100) -> torch.Tensor:
    """METIS text of a device DAG (header included) as a uint8 device tensor."""
    from .kway import in_order, symmetrize
    fn = _native._need(_emit, "hs_emit_metis")
    w_node = csr.w_gpu if node_weight_source == GPU else csr.w_cpu
    r = csr.root
    if r < 0:
        raise PartitionError("graph has no root node; cannot export kernels")
    # K1 lowers kernels by dropping the root's out-list; an edge INTO the root
    # (a cyclic, never-validated graph) has no place in that layout
    if int(csr.in_ptr[r + 1] - csr.in_ptr[r]) != 0:
        raise PartitionError("graph has edges into the root; validate() it before export")
    inter = torch.ones(csr.m, dtype=torch.bool, device=csr.device)
    inter[int(csr.out_ptr[r]):int(csr.out_ptr[r + 1])] = False  # root edges
    kern = torch.ones(csr.n, dtype=torch.bool, device=csr.device)
    kern[r] = False
    if bool((w_node[kern] == 0).all()) and bool((csr.w_xfer[inter] == 0).all()):
        raise PartitionError("all weights are zero; cannot integerize for export")
    ew = _scaled(csr.w_xfer, scale)
    ug = symmetrize(csr, ew, _scaled(w_node, scale), in_order(csr, ew), unit_ok=False)
    n_inter = int(inter.sum().item())
    header = f"{ug.n} {n_inter} 011\n".encode()
    size = ctypes.c_int64(0)
    _native.check(fn(ctypes.byref(ug.struct()), None, 0, ctypes.byref(size),
                     _native.stream_ptr()))
    out = torch.empty(len(header) + size.value, dtype=torch.uint8, device=csr.device)
    out[:len(header)] = torch.frombuffer(bytearray(header), dtype=torch.uint8).to(csr.device)
    _native.check(fn(ctypes.byref(ug.struct()), out.data_ptr() + len(header), size.value,
                     ctypes.byref(size), _native.stream_ptr()))
    return out


def emit_metis(graph: TaskGraph, node_weight_source: str = GPU, scale: int = 100) -> str:
    """graphio.py:277-304 — the kernels as an undirected METIS graph, on the device."""
    text = emit_metis_csr(graph.csr(), node_weight_source, scale)
    return bytes(text.cpu().numpy()).decode("ascii")


def parse_partition_bytes(data, n_expected: int,
                          device=None) -> Tuple[Optional[torch.Tensor], Optional[str]]:
    """Device parse of a METIS partition file: (int8 [n_expected] groups, None) or
    (None, the reference's error message)."""
    fn = _native._need(_parse, "hs_parse_partition")
    dev = device or _native.device()
    raw = data.encode("utf-8") if isinstance(data, str) else bytes(data)
    buf = torch.frombuffer(bytearray(raw), dtype=torch.uint8).to(dev) if raw else \
        torch.empty(1, dtype=torch.uint8, device=dev)
    part = torch.zeros(max(n_expected, 1), dtype=torch.int8, device=dev)
    cap = 64
    while True:
        odd = (ctypes.c_int64 * (3 * cap))()
        vals = (ctypes.c_int64 * cap)()
        info = (ctypes.c_int64 * 4)()
        _native.check(fn(buf.data_ptr(), len(raw), int(n_expected), part.data_ptr(), odd, vals,
                         cap, info, _native.stream_ptr()))
        if info[1] <= cap:
            break
        cap = int(info[1])
    n_lines = info[0]
    fixes = []
    text = None
    for i in range(info[1]):
        line_idx, cls, slot = odd[3 * i], odd[3 * i + 1], odd[3 * i + 2]
        lineno = line_idx + 1
        if cls == 3:  # a plain integer other than 0/1 (graphio.py:323-324)
            return None, f"line {lineno}: group must be 0 or 1, got {vals[i]}"
        # undecided on the device: Python's own int() on that one line
        if text is None:
            text = raw.decode("utf-8").splitlines()
        line = text[line_idx].strip()
        try:
            v = int(line)
        except ValueError:
            return None, f"line {lineno}: not an integer: {line!r}"
        if v not in (0, 1):
            return None, f"line {lineno}: group must be 0 or 1, got {v}"
        fixes.append((slot, v))
    if n_lines != n_expected:
        return None, f"partition file has {n_lines} lines for {n_expected} kernels"
    if fixes:
        idx = torch.tensor([s for s, _ in fixes], dtype=torch.int64, device=dev)
        part[idx] = torch.tensor([v for _, v in fixes], dtype=torch.int8, device=dev)
    return part[:n_expected], None


def parse_partition_file(text: str, graph: TaskGraph, targets: Optional[PartitionTargets] = None,
                         node_weight_source: str = GPU, tolerance: float = 0.03) -> Partition:
    """graphio.py:307-330 — read a METIS partition file (one 0/1 line per kernel)."""
    ids = graph.kernel_ids()
    part, err = parse_partition_bytes(text, len(ids))
    if err is not None:
        raise PartitionError(err)
    groups = part.cpu().numpy()
    assignment = {nid: (CPU if g == 0 else GPU) for nid, g in zip(ids, groups.tolist())}
    if targets is None:
        from .costs import workload_ratio
        targets = workload_ratio(graph)
    return _finish(graph, assignment, targets, node_weight_source, tolerance)


def emit_partition_file(partition: Partition, graph: TaskGraph) -> str:
    """graphio.py:333-339 — inverse of parse_partition_file (0 = CPU, 1 = GPU)."""
    return "".join("0\n" if partition.assignment[nid] == CPU else "1\n"
                   for nid in graph.kernel_ids())


def emit_partition_bytes(part: torch.Tensor) -> torch.Tensor:
    """Device form of emit_partition_file for a 0/1 part array: '0\\n'/'1\\n' per kernel."""
    p = part.to(torch.uint8)
    out = torch.empty(2 * p.numel(), dtype=torch.uint8, device=p.device)
    out[0::2] = p + ord("0")
    out[1::2] = ord("\n")
    return out
