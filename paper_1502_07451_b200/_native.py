"""ctypes binding of the C ABI in include/hetsched_b200.h (libhetsched_b200.so).

This module is the only place the package touches the native library. There
is no CPU fallback: importing it without the built library raises, and every
call requires a CUDA device. Device buffers are torch CUDA tensors (torch is
the allocator/stream plumbing only); calls run on torch's current stream.
"""
from __future__ import annotations

import ctypes
import os
import warnings
from typing import Optional, Tuple

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libhetsched_b200.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `make` (or __graft_entry__.build()). "
        "The hot path has no CPU fallback.")
_lib = ctypes.CDLL(LIB_PATH)

HS_EDEADLOCK = -5
_c_void_p = ctypes.c_void_p
_i32, _i64, _f64 = ctypes.c_int32, ctypes.c_int64, ctypes.c_double


class NativeError(RuntimeError):
    def __init__(self, code: int, message: str):
        super().__init__(f"hetsched_b200 error {code}: {message}")
        self.code = code
        self.message = message


class HsDag(ctypes.Structure):
    _fields_ = [("n", _i32), ("root", _i32), ("m", _i64),
                ("out_ptr", _c_void_p), ("out_dst", _c_void_p),
                ("in_ptr", _c_void_p), ("in_src", _c_void_p), ("in_eid", _c_void_p),
                ("w_cpu", _c_void_p), ("w_gpu", _c_void_p),
                ("w_xfer", _c_void_p), ("bytes", _c_void_p)]


class HsDagBatch(ctypes.Structure):
    _fields_ = [("batch", _i32), ("total_nodes", _i64), ("total_edges", _i64),
                ("node_off", _c_void_p), ("edge_off", _c_void_p), ("root", _c_void_p),
                ("out_ptr", _c_void_p), ("out_dst", _c_void_p),
                ("in_ptr", _c_void_p), ("in_src", _c_void_p), ("in_eid", _c_void_p),
                ("w_cpu", _c_void_p), ("w_gpu", _c_void_p),
                ("w_xfer", _c_void_p), ("bytes", _c_void_p)]


class HsUGraph(ctypes.Structure):
    _fields_ = [("n", _i32), ("nnz", _i64), ("xadj", _c_void_p), ("adjncy", _c_void_p),
                ("adjwgt", _c_void_p), ("adjwgt_i", _c_void_p),
                ("vwgt", _c_void_p), ("vwgt_i", _c_void_p), ("twin", _c_void_p)]


class HsDist(ctypes.Structure):
    _fields_ = [("rank", _i32), ("size", _i32), ("arena", _c_void_p * 8), ("arena_bytes", _i64),
                ("mode", _i32)]


class HsEvent(ctypes.Structure):
    _fields_ = [("time", _f64), ("kind", _i32), ("a", _i32), ("b", _i32),
                ("resource", _i32)]


EVENT_DTYPE = np.dtype([("time", "<f8"), ("kind", "<i4"), ("a", "<i4"), ("b", "<i4"),
                        ("resource", "<i4")])
assert EVENT_DTYPE.itemsize == ctypes.sizeof(HsEvent)


def _proto(name, *argtypes):
    fn = getattr(_lib, name)
    fn.restype = ctypes.c_int
    fn.argtypes = list(argtypes)
    return fn


_P = _c_void_p
_lib.hs_last_error.restype = ctypes.c_char_p
_lib.hs_version.restype = ctypes.c_char_p
_lib.hs_launch_count.restype = ctypes.c_int64
_exact_totals = _proto("hs_exact_totals", _P, ctypes.c_int, _P, _P)
_evaluate2 = _proto("hs_evaluate2", _P, _P, _i32, ctypes.c_int, ctypes.c_int, _P, _P, _P, _P)
_evaluate_kway = _proto("hs_evaluate_kway", _P, _P, _i32, _i32, _P, _P, _P, _P, _P, _P, _P)
_levels = _proto("hs_levels", _P, ctypes.c_int, _P, _P, _P, _P, _P)
_level_order = _proto("hs_level_order", _P, _P, _i32, _P, _P)
_simulate_batch = _proto("hs_simulate_batch", _P, ctypes.c_int, _P, _i32, _i32,
                         _P, _P, _P, _P, _P, _P, _P, _P, _P, _P)


def _opt(name, *argtypes):
    return _proto(name, *argtypes) if hasattr(_lib, name) else None


_fm2 = _opt("hs_fm2", _P, _P, _P, _P, _i64, _P, _f64, _f64, _P, _i32, _P, _P, _P, _P, _P)
_brute2 = _opt("hs_brute2", _i32, _P, _f64, _f64, _P, _P, _P, _i64, _P, _P, _P)
_partition_kway = _opt("hs_partition_kway", _P, _i32, _P, _f64, ctypes.c_uint64, _P, _P, _P)
_symmetrize = _opt("hs_symmetrize", _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P)
_symmetrize_range = _opt("hs_symmetrize_range", _P, _i32, _i32, _P, _P, _P, _P, _P, _P, _P, _P,
                         _P, _P)
_dag_transpose = _opt("hs_dag_transpose", _i32, _i64, _P, _P, _P, _P, _P, _P)
_int32_stats = _opt("hs_int32_stats", _P, _i64, _P, _P)
_integer_weights = _opt("hs_integer_weights", _P, _i64, _i32, _P, _P)
_partition_kway_dist = _opt("hs_partition_kway_dist", _P, _i32, _i32, _P, _i32, _P, _f64,
                            ctypes.c_uint64, _P, _P, _P)
if hasattr(_lib, "hs_kway_dist_arena_bytes"):
    _lib.hs_kway_dist_arena_bytes.restype = ctypes.c_int64
    _lib.hs_kway_dist_arena_bytes.argtypes = [_i32]
_layered_sizes = _opt("hs_layered_sizes", _i64, _i64, _P, _P)
_layered_generate = _opt("hs_layered_generate", _i64, _i64, ctypes.c_uint64,
                         _P, _P, _P, _P, _P, _P, _P)


def version() -> str:
    return _lib.hs_version().decode()


def launch_count() -> int:
    return int(_lib.hs_launch_count())


def check(rc: int) -> None:
    if rc != 0:
        raise NativeError(rc, _lib.hs_last_error().decode(errors="replace"))


def device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("hetsched_b200 needs a CUDA device (sm_100a); "
                           "there is no CPU fallback on the hot path")
    return torch.device("cuda", torch.cuda.current_device())


def stream_ptr() -> int:
    return torch.cuda.current_stream().cuda_stream


def ptr(t: Optional[torch.Tensor]) -> Optional[int]:
    if t is None:
        return None
    assert t.is_cuda and t.is_contiguous(), "device tensors must be contiguous CUDA tensors"
    return t.data_ptr()


def _need(fn, name):
    if fn is None:
        raise NativeError(-1, f"{name} is not exported by {LIB_PATH}")
    return fn


# ---------------------------------------------------------------- wrappers --

def exact_totals(csr, include_root: bool) -> Tuple[float, float, float]:
    out = (ctypes.c_double * 3)()
    check(_exact_totals(ctypes.byref(csr.struct()), int(include_root), out, stream_ptr()))
    return out[0], out[1], out[2]


def evaluate2(csr, parts: torch.Tensor, weight_source: int, mode: int):
    """parts: int8 [B, n_kernels] device tensor. Returns (cut, cpu_w, total) f64 [B]."""
    b = parts.shape[0]
    dev = parts.device
    cut = torch.empty(b, dtype=torch.float64, device=dev)
    cpu_w = torch.empty_like(cut)
    total = torch.empty_like(cut)
    check(_evaluate2(ctypes.byref(csr.struct()), ptr(parts), b, weight_source, mode,
                     ptr(cut), ptr(cpu_w), ptr(total), stream_ptr()))
    return cut, cpu_w, total


def evaluate_kway(csr, parts: torch.Tensor, k: int, vwgt_i: torch.Tensor):
    """parts: int32 [B, n] (node index space). Returns dict of int64 tensors."""
    b = parts.shape[0]
    dev = parts.device
    z = lambda *s: torch.empty(*s, dtype=torch.int64, device=dev)  # noqa: E731
    out = dict(cut_bytes=z(b), cut_edges=z(b), loads=z(b, k), xfer_count=z(b),
               xfer_bytes=z(b))
    check(_evaluate_kway(ctypes.byref(csr.struct()), ptr(parts), b, k, ptr(vwgt_i),
                         ptr(out["cut_bytes"]), ptr(out["cut_edges"]), ptr(out["loads"]),
                         ptr(out["xfer_count"]), ptr(out["xfer_bytes"]), stream_ptr()))
    return out


def levels(csr, mode: int = 0, sync: bool = True):
    dev = csr.device
    level = torch.empty(csr.n, dtype=torch.int32, device=dev)
    finish = torch.empty(csr.n, dtype=torch.float64, device=dev)
    cp = ctypes.c_double(0.0)
    nl = ctypes.c_int32(0)
    check(_levels(ctypes.byref(csr.struct()), mode, ptr(level), ptr(finish),
                  ctypes.byref(cp) if sync else None, ctypes.byref(nl) if sync else None,
                  stream_ptr()))
    return level, finish, cp.value, nl.value


_assigned_makespan = _opt("hs_assigned_makespan", _P, _P, _P, _i32, _P, _P, _P, _P)


def assigned_makespan(csr, part: torch.Tensor, dev: torch.Tensor):
    """(makespan, finish f64 [n]) of a node-space assignment (hs_assigned_makespan)."""
    fn = _need(_assigned_makespan, "hs_assigned_makespan")
    level = torch.empty(csr.n, dtype=torch.int32, device=csr.device)
    finish = torch.empty(csr.n, dtype=torch.float64, device=csr.device)
    ms = ctypes.c_double(0.0)
    check(fn(ctypes.byref(csr.struct()), ptr(part), ptr(dev), int(dev.numel()), ptr(level),
             ptr(finish), ctypes.byref(ms), stream_ptr()))
    return ms.value, finish


def level_order(csr, level: torch.Tensor, n_levels: int) -> torch.Tensor:
    order = torch.empty(csr.n, dtype=torch.int32, device=csr.device)
    check(_level_order(ctypes.byref(csr.struct()), ptr(level), n_levels, ptr(order),
                       stream_ptr()))
    return order


_is_topological = _opt("hs_dag_is_topological", _P, _P, _P)
_topo_order = _opt("hs_topological_order", _P, _P, _P, _P, _P, _P)


def topological_order(csr):
    """(order int32 [n] device, count, stuck index or -1, rounds) — hs_topological_order."""
    order = torch.empty(max(csr.n, 1), dtype=torch.int32, device=csr.device)
    cnt, stuck, rounds = ctypes.c_int32(0), ctypes.c_int32(-1), ctypes.c_int32(0)
    check(_need(_topo_order, "hs_topological_order")(
        ctypes.byref(csr.struct()), ptr(order), ctypes.byref(cnt), ctypes.byref(stuck),
        ctypes.byref(rounds), stream_ptr()))
    return order[:csr.n], cnt.value, stuck.value, rounds.value
_level_permutation = _opt("hs_level_permutation", _P, _P, _i32, _P, _P, _P)
_ugraph_permute = _opt("hs_ugraph_permute", _P, _P, _P, _P, _P, _P, _P, _P)
_parts_unpermute = _opt("hs_parts_unpermute", _i32, _P, _P, _P, _P)


def dag_is_topological(csr) -> bool:
    out = ctypes.c_int32(0)
    check(_need(_is_topological, "hs_dag_is_topological")(ctypes.byref(csr.struct()),
                                                          ctypes.byref(out), stream_ptr()))
    return bool(out.value)


def level_permutation(csr, level: torch.Tensor, n_levels: int):
    nk = csr.n - 1
    perm = torch.empty(nk, dtype=torch.int32, device=csr.device)
    inv = torch.empty(nk, dtype=torch.int32, device=csr.device)
    check(_need(_level_permutation, "hs_level_permutation")(
        ctypes.byref(csr.struct()), ptr(level), n_levels, ptr(perm), ptr(inv), stream_ptr()))
    return perm, inv


def ugraph_permute(ug, perm: torch.Tensor, inv: torch.Tensor):
    """(xadj, adjncy, adjwgt or None, vwgt) of the relabelled graph."""
    dev = ug.xadj.device
    xadj = torch.empty(ug.n + 1, dtype=torch.int64, device=dev)
    adjncy = torch.empty(ug.nnz, dtype=torch.int32, device=dev)
    adjwgt = (torch.empty(ug.nnz, dtype=torch.int32, device=dev)
              if ug._adjwgt is not None else None)
    vwgt = torch.empty(ug.n, dtype=torch.int32, device=dev)
    check(_need(_ugraph_permute, "hs_ugraph_permute")(
        ctypes.byref(ug.struct()), ptr(perm), ptr(inv), ptr(xadj), ptr(adjncy),
        ptr(adjwgt) if adjwgt is not None else None, ptr(vwgt), stream_ptr()))
    return xadj, adjncy, adjwgt, vwgt


def parts_unpermute(perm: torch.Tensor, part_new: torch.Tensor, out: torch.Tensor):
    check(_need(_parts_unpermute, "hs_parts_unpermute")(int(perm.numel()), ptr(perm),
                                                        ptr(part_new), ptr(out), stream_ptr()))
    return out


def simulate_batch(batch, policy: int, pin: Optional[torch.Tensor], cpu_workers: int,
                   gpu_workers: int, events: bool = False):
    """Runs batch.batch simulations; returns a dict of device tensors."""
    b = batch.batch
    dev = batch.device
    out = dict(
        makespan=torch.empty(b, dtype=torch.float64, device=dev),
        transfer_count=torch.empty(b, dtype=torch.int64, device=dev),
        transfer_bytes=torch.empty(b, dtype=torch.int64, device=dev),
        busy=torch.empty(b, 2, dtype=torch.float64, device=dev),
        kpd=torch.empty(b, 2, dtype=torch.int64, device=dev),
        status=torch.empty(b, dtype=torch.int32, device=dev),
    )
    ev = ev_off = ev_count = None
    if events:
        cap = 2 * (batch.node_counts + batch.edge_counts)
        ev_off_h = np.zeros(b + 1, dtype=np.int64)
        np.cumsum(cap, out=ev_off_h[1:])
        ev_off = torch.from_numpy(ev_off_h).to(dev)
        ev = torch.empty(int(ev_off_h[-1]) * EVENT_DTYPE.itemsize, dtype=torch.uint8, device=dev)
        ev_count = torch.empty(b, dtype=torch.int64, device=dev)
        out.update(events=ev, ev_off=ev_off, ev_count=ev_count)
    check(_simulate_batch(ctypes.byref(batch.struct()), policy, ptr(pin), cpu_workers,
                          gpu_workers, ptr(out["makespan"]), ptr(out["transfer_count"]),
                          ptr(out["transfer_bytes"]), ptr(out["busy"]), ptr(out["kpd"]),
                          ptr(out["status"]), ptr(ev), ptr(ev_off), ptr(ev_count),
                          stream_ptr()))
    return out


class HsCostTable(ctypes.Structure):
    _fields_ = [("n_pairs", ctypes.c_int32), ("form", _P), ("cpu", _P), ("gpu", _P),
                ("ma_cpu", ctypes.c_double), ("ma_gpu", ctypes.c_double),
                ("mm_cpu", ctypes.c_double), ("mm_gpu", ctypes.c_double),
                ("launch_ms", ctypes.c_double), ("latency_ms", ctypes.c_double),
                ("bandwidth", ctypes.c_double)]


_attach = _opt("hs_attach_weights", _P, _i32, _P, _P, _P, _P, _P, ctypes.c_int64, _P, _P, _P,
               _P, _P, _P)


def attach_weights(form, cpu, gpu, transfer, pair, size, rank, nbytes, xfer_tab, dev):
    """(w_cpu, w_gpu, w_xfer, bad_node_rank, bad_edge) — hs_attach_weights."""
    from . import costs as C
    f = torch.tensor(form or [0], dtype=torch.int32, device=dev)
    c = torch.tensor(cpu or [0.0], dtype=torch.float64, device=dev)
    g = torch.tensor(gpu or [0.0], dtype=torch.float64, device=dev)
    t = HsCostTable(len(form), ptr(f), ptr(c), ptr(g), C.MA_CPU_COEFF, C.MA_GPU_COEFF,
                    C.MM_CPU_COEFF, C.MM_GPU_COEFF, C.GPU_LAUNCH_MS,
                    transfer.latency_ms if transfer is not None else 0.0,
                    transfer.bandwidth_bytes_per_ms if transfer is not None else 1.0)
    n, m = int(pair.numel()), int(nbytes.numel())
    w_cpu = torch.empty(n, dtype=torch.float64, device=dev)
    w_gpu = torch.empty(n, dtype=torch.float64, device=dev)
    w_xfer = torch.empty(m, dtype=torch.float64, device=dev)
    bn, be = ctypes.c_int32(-1), ctypes.c_int64(-1)
    check(_need(_attach, "hs_attach_weights")(ctypes.byref(t), n, ptr(pair), ptr(size), ptr(rank),
                                              ptr(w_cpu), ptr(w_gpu), m, ptr(nbytes),
                                              ptr(xfer_tab), ptr(w_xfer), ctypes.byref(bn),
                                              ctypes.byref(be), stream_ptr()))
    return w_cpu, w_gpu, w_xfer, bn.value, be.value


_rgen = _opt("hs_random_dag_batch", _i32, _P, _i32, _i32, _P, ctypes.c_int64, ctypes.c_int64,
             ctypes.c_int64, _i32, ctypes.c_int64, ctypes.c_int64, _P, _P, _P, _P, _P, _P,
             ctypes.c_int64, _P)


def random_dag_batch(seeds: torch.Tensor, shape: dict, n_nodes: int):
    """(edge_counts, out_ptr, out_dst, in_ptr, in_src, in_eid) of hs_random_dag_batch."""
    fn = _need(_rgen, "hs_random_dag_batch")
    b = int(seeds.numel())
    dev = seeds.device
    first = torch.tensor(shape["first"], dtype=torch.int32, device=dev)
    counts = (ctypes.c_int64 * max(b, 1))()
    args = (b, ptr(seeds), shape["n_real"], shape["n_layers"], ptr(first), shape["base_capacity"],
            shape["inter_target"], shape["extra"], shape["mode"], shape["pop_cap"],
            shape["edge_cap"], counts)
    check(fn(*args, None, None, None, None, None, 0, stream_ptr()))
    m = np.frombuffer(counts, dtype=np.int64, count=b).copy()
    total = int(m.sum())
    out_ptr = torch.empty(b * (n_nodes + 1), dtype=torch.int64, device=dev)
    in_ptr = torch.empty(b * (n_nodes + 1), dtype=torch.int64, device=dev)
    out_dst = torch.empty(max(total, 1), dtype=torch.int32, device=dev)
    in_src = torch.empty(max(total, 1), dtype=torch.int32, device=dev)
    in_eid = torch.empty(max(total, 1), dtype=torch.int32, device=dev)
    check(fn(*args, ptr(out_ptr), ptr(out_dst), ptr(in_ptr), ptr(in_src), ptr(in_eid), total,
             stream_ptr()))
    return m, out_ptr, out_dst[:total], in_ptr, in_src[:total], in_eid[:total]


_trace_sort = _opt("hs_trace_sort", _P, ctypes.c_int64, _P, _P, _P, _P)
_trace_metrics = _opt("hs_trace_metrics", _P, _P, ctypes.c_int64, _i32, _i32, _P, _P)


def trace_sort(ev: torch.Tensor, count: int, ids: torch.Tensor, res_rank: torch.Tensor
               ) -> torch.Tensor:
    """perm[count]: the reference's event order (hs_trace_sort); ev is a uint8
    view of count hs_event_t records."""
    perm = torch.empty(max(count, 1), dtype=torch.int32, device=ids.device)
    check(_need(_trace_sort, "hs_trace_sort")(ptr(ev), count, ptr(ids), ptr(res_rank),
                                              ptr(perm), stream_ptr()))
    return perm[:count]


def trace_metrics(ev: torch.Tensor, perm: torch.Tensor, count: int, n_nodes: int,
                  cpu_workers: int):
    """(makespan, transfers, busy_cpu, busy_gpu, kernels_cpu, kernels_gpu) — hs_trace_metrics."""
    out = (ctypes.c_double * 6)()
    check(_need(_trace_metrics, "hs_trace_metrics")(ptr(ev), ptr(perm), count, n_nodes,
                                                    cpu_workers, out, stream_ptr()))
    return tuple(out)


def fm2(ug, edge_w, edge_u, edge_v, weights, r_cpu, tol, orders, start):
    fn = _need(_fm2, "hs_fm2")
    n_orders = orders.shape[0]
    dev = weights.device
    assign = torch.empty(n_orders, ug.n, dtype=torch.int8, device=dev)
    cut = torch.empty(n_orders, dtype=torch.float64, device=dev)
    err = torch.empty(n_orders, dtype=torch.float64, device=dev)
    check(fn(ctypes.byref(ug.struct()), ptr(edge_w), ptr(edge_u), ptr(edge_v),
             int(edge_w.numel()), ptr(weights), float(r_cpu), float(tol), ptr(orders),
             n_orders, ptr(start), ptr(assign), ptr(cut), ptr(err), stream_ptr()))
    return assign, cut, err


def brute2(n, weights, r_cpu, tol, edge_a, edge_b, edge_w):
    fn = _need(_brute2, "hs_brute2")
    mask = ctypes.c_int64(0)
    feas = ctypes.c_int32(0)
    check(fn(n, ptr(weights), float(r_cpu), float(tol), ptr(edge_a), ptr(edge_b),
             ptr(edge_w), int(edge_w.numel()), ctypes.byref(mask), ctypes.byref(feas),
             stream_ptr()))
    return mask.value, bool(feas.value)


_partition_kway_starts = _opt("hs_partition_kway_starts", _P, _i32, _P, ctypes.c_double,
                              ctypes.c_uint64, _P, _i32, _P, _P, _P)


def partition_kway(ug, k: int, tpwgts, tol: float, seed: int, part: torch.Tensor,
                   starts: Optional[torch.Tensor] = None):
    """hs_partition_kway, or hs_partition_kway_starts with int32 [S, n] device starts."""
    tp = (ctypes.c_double * k)(*[float(x) for x in tpwgts])
    stats = (ctypes.c_int64 * 8)()
    sd = ctypes.c_uint64(seed & (2**64 - 1))
    if starts is not None and starts.shape[0] > 0:
        fn = _need(_partition_kway_starts, "hs_partition_kway_starts")
        check(fn(ctypes.byref(ug.struct()), k, tp, float(tol), sd, ptr(starts),
                 int(starts.shape[0]), ptr(part), stats, stream_ptr()))
    else:
        fn = _need(_partition_kway, "hs_partition_kway")
        check(fn(ctypes.byref(ug.struct()), k, tp, float(tol), sd, ptr(part), stats,
                 stream_ptr()))
    return list(stats)


def dag_transpose(n: int, m: int, out_ptr, out_dst, in_ptr, in_src, in_eid) -> None:
    fn = _need(_dag_transpose, "hs_dag_transpose")
    check(fn(n, m, ptr(out_ptr), ptr(out_dst), ptr(in_ptr), ptr(in_src), ptr(in_eid),
             stream_ptr()))


def int32_stats(t: torch.Tensor) -> Tuple[int, int, int]:
    """(sum, min, max) of an int32 device tensor (hs_int32_stats)."""
    fn = _need(_int32_stats, "hs_int32_stats")
    out = (ctypes.c_int64 * 3)()
    check(fn(ptr(t), t.numel(), out, stream_ptr()))
    return out[0], out[1], out[2]


def integer_weights(w: torch.Tensor, scale: int) -> torch.Tensor:
    """max(1, floor(w * scale + 0.5)) as int32 on the device (hs_integer_weights)."""
    fn = _need(_integer_weights, "hs_integer_weights")
    w = w.contiguous()
    if w.dtype != torch.float64 or not w.is_cuda:
        raise TypeError("integer_weights: fp64 device tensor expected")
    out = torch.empty(w.shape, dtype=torch.int32, device=w.device)
    check(fn(ptr(w), w.numel(), int(scale), ptr(out), stream_ptr()))
    return out


def symmetrize(csr, edge_w_i, node_w_i, xadj, adjncy, adjwgt_i, vwgt_i, edge_w_i_in=None,
               twin=None, read_nnz: bool = True) -> int:
    """read_nnz=False: no host read of the entry count (returns -1; the caller knows it)."""
    fn = _need(_symmetrize, "hs_symmetrize")
    nnz = ctypes.c_int64(-1)
    check(fn(ctypes.byref(csr.struct()), ptr(edge_w_i), ptr(edge_w_i_in), ptr(node_w_i), ptr(xadj),
             ptr(adjncy), ptr(adjwgt_i), ptr(vwgt_i), ptr(twin),
             ctypes.byref(nnz) if read_nnz else None, stream_ptr()))
    return nnz.value


def symmetrize_range(csr, kv0: int, kv1: int, edge_w_i, node_w_i, xadj, adjncy, adjwgt_i,
                     vwgt_i, edge_w_i_in=None) -> int:
    fn = _need(_symmetrize_range, "hs_symmetrize_range")
    nnz = ctypes.c_int64(0)
    check(fn(ctypes.byref(csr.struct()), kv0, kv1, ptr(edge_w_i), ptr(edge_w_i_in),
             ptr(node_w_i), ptr(xadj), ptr(adjncy), ptr(adjwgt_i), ptr(vwgt_i), None,
             ctypes.byref(nnz), stream_ptr()))
    return nnz.value


_validate_dag = _opt("hs_validate_dag", _P, _P, _P, _P, _P, _P)


def validate_dag(csr, node_bad: Optional[torch.Tensor] = None,
                 edge_bad: Optional[torch.Tensor] = None):
    """(counts[7], first[7]) of the device validation checks (hs_validate_dag)."""
    fn = _need(_validate_dag, "hs_validate_dag")
    counts = (ctypes.c_int64 * 7)()
    first = (ctypes.c_int32 * 7)()
    check(fn(ctypes.byref(csr.struct()), counts, first, ptr(node_bad), ptr(edge_bad),
             stream_ptr()))
    return list(counts), list(first)


def kway_dist_arena_bytes(n_global: int) -> int:
    return int(_lib.hs_kway_dist_arena_bytes(n_global))


def partition_kway_dist(ug, v0: int, n_global: int, dist: HsDist, k: int, tpwgts, tol: float,
                        seed: int, part: torch.Tensor):
    """One rank's call (blocks until every rank of the group has made its own)."""
    fn = _need(_partition_kway_dist, "hs_partition_kway_dist")
    tp = (ctypes.c_double * k)(*[float(x) for x in tpwgts])
    stats = (ctypes.c_int64 * 8)()
    check(fn(ctypes.byref(ug.struct()), v0, n_global, ctypes.byref(dist), k, tp, float(tol),
             ctypes.c_uint64(seed & (2**64 - 1)), ptr(part), stats, stream_ptr()))
    return list(stats)


def layered_sizes(n_kernels: int, m_inter: int) -> Tuple[int, int]:
    fn = _need(_layered_sizes, "hs_layered_sizes")
    n, m = ctypes.c_int64(0), ctypes.c_int64(0)
    check(fn(n_kernels, m_inter, ctypes.byref(n), ctypes.byref(m)))
    return n.value, m.value


def layered_generate(n_kernels, m_inter, seed, out_ptr, out_dst, in_ptr, in_src, in_eid,
                     layer_of):
    fn = _need(_layered_generate, "hs_layered_generate")
    check(fn(n_kernels, m_inter, ctypes.c_uint64(seed & (2**64 - 1)), ptr(out_ptr),
             ptr(out_dst), ptr(in_ptr), ptr(in_src), ptr(in_eid), ptr(layer_of),
             stream_ptr()))


# ---------------------------------------------------------------- profiling --
_lib.hs_profile_enable.argtypes = [ctypes.c_int]
_lib.hs_profile_enable.restype = None
_lib.hs_profile_reset.restype = None
_lib.hs_profile_report.argtypes = [ctypes.c_char_p, ctypes.c_int]
_lib.hs_profile_report.restype = ctypes.c_int


def profile_enable(on: bool = True) -> None:
    _lib.hs_profile_enable(1 if on else 0)


def profile_reset() -> None:
    _lib.hs_profile_reset()


def profile_report() -> dict:
    """{kernel: {"launches", "ms", "bytes"}} accumulated since the last reset."""
    size = _lib.hs_profile_report(None, 0)
    buf = ctypes.create_string_buffer(size + 1)
    _lib.hs_profile_report(buf, size + 1)
    out = {}
    for line in buf.value.decode().splitlines():
        name, launches, ms, nbytes = line.split(",")
        out[name] = {"launches": int(launches), "ms": float(ms), "bytes": float(nbytes)}
    return out


_fm2_batch = _opt("hs_fm2_batch", _i32, _P, _P, _P, _i64, _i32, _P, _P, _P, _P, _P, _P, _P, _P, _f64,
                  _P, _i32, _P, _P, _P, _P, _P)
_exact_totals_batch = _opt("hs_exact_totals_batch", _P, ctypes.c_int, _P, _P)


_gp_pins = _opt("hs_gp_pins_batch", _P, _i32, _P, _i32, ctypes.c_double, _P, _P, _P)


def gp_pins_batch(batch, restarts: int, shuffles: Optional[torch.Tensor], n_shuffle: int,
                  tol: float):
    """(pin int8 [total nodes], flags np.int32 [G]) — hs_gp_pins_batch."""
    pin = torch.empty(max(int(batch.node_off_h[-1]), 1), dtype=torch.int8, device=batch.device)
    flags = np.zeros(max(batch.batch, 1), dtype=np.int32)
    check(_need(_gp_pins, "hs_gp_pins_batch")(
        ctypes.byref(batch.struct()), restarts, ptr(shuffles), n_shuffle, float(tol), ptr(pin),
        flags.ctypes.data_as(ctypes.c_void_p), stream_ptr()))
    return pin[:int(batch.node_off_h[-1])], flags[:batch.batch]


def fm2_batch(tb, weights, r_cpu, tol, orders, n_orders):
    """Batched exact 2-way partitioner; returns (assign int8 flat, cut [G,R], err [G,R], status)."""
    fn = _need(_fm2_batch, "hs_fm2_batch")
    dev = weights.device
    G = tb.G
    assign = torch.empty(n_orders * tb.total_nodes, dtype=torch.int8, device=dev)
    cut = torch.empty(G, n_orders, dtype=torch.float64, device=dev)
    err = torch.empty(G, n_orders, dtype=torch.float64, device=dev)
    status = torch.zeros(G, n_orders, dtype=torch.int32, device=dev)
    check(fn(G, ptr(tb.node_off), ptr(tb.adj_off), ptr(tb.edge_off), tb.total_nodes, tb.max_n,
             ptr(tb.xadj), ptr(tb.adjncy), ptr(tb.adjwgt), ptr(tb.edge_w), ptr(tb.edge_u),
             ptr(tb.edge_v), ptr(weights), ptr(r_cpu), float(tol), ptr(orders), n_orders,
             ptr(assign), ptr(cut), ptr(err), ptr(status), stream_ptr()))
    return assign, cut, err, status


def exact_totals_batch(batch, include_root: bool) -> torch.Tensor:
    fn = _need(_exact_totals_batch, "hs_exact_totals_batch")
    out = torch.empty(batch.batch, 3, dtype=torch.float64, device=batch.device)
    check(fn(ctypes.byref(batch.struct()), int(include_root), ptr(out), stream_ptr()))
    return out


# ---- DOT ingestion (hs_dot_*) ------------------------------------------------
class HsDotInfo(ctypes.Structure):
    _fields_ = [("status", _i32), ("err_line", _i32), ("err_a", _i32), ("err_b", _i32),
                ("err_c", _i32), ("name_b", _i32), ("name_e", _i32), ("n_names", _i32),
                ("n_edges", _i32), ("n_attrs", _i32), ("n_slow", _i32), ("root_rank", _i32),
                ("conv_err", _i64), ("max_id", _i64)]


class HsDotHost(ctypes.Structure):
    _fields_ = [(f, _c_void_p) for f in (
        "id", "kind_attr", "kind_hash", "size", "w_cpu", "w_gpu", "has_pred",
        "src", "dst", "bytes", "w_xfer", "k0", "k1", "v0", "v1", "owner", "cls", "slow")]


_dot_parse = _opt("hs_dot_parse", _P, _i64, _P, _P, _P)
_dot_fetch = _opt("hs_dot_fetch", _P, _P, _P)
_dot_csr_size = _opt("hs_dot_csr_size", _P, _P, _P, _P)
_dot_csr = _opt("hs_dot_csr", _P, _P, _P, _P, _P, _P, _P, _P, _P, _P)
_dot_release = _opt("hs_dot_release", _P)
_dot_py_float = _opt("hs_dot_py_float", ctypes.c_char_p, _i64, _P)

_DOT_FIELDS = {  # field -> (dtype, count key)
    "id": (np.int64, "n_names"), "kind_attr": (np.int32, "n_names"),
    "kind_hash": (np.uint64, "n_names"), "size": (np.int64, "n_names"),
    "w_cpu": (np.float64, "n_names"), "w_gpu": (np.float64, "n_names"),
    "has_pred": (np.uint8, "n_names"), "src": (np.int32, "n_edges"),
    "dst": (np.int32, "n_edges"), "bytes": (np.int64, "n_edges"),
    "w_xfer": (np.float64, "n_edges"), "k0": (np.int32, "n_attrs"),
    "k1": (np.int32, "n_attrs"), "v0": (np.int32, "n_attrs"), "v1": (np.int32, "n_attrs"),
    "owner": (np.int32, "n_attrs"), "cls": (np.uint8, "n_attrs"),
}


class DotHandle:
    """A device parse (hs_dot_parse); released when collected or by ``close``."""

    def __init__(self, text_dev: torch.Tensor, info: HsDotInfo, handle: int):
        self.text_dev = text_dev  # the parse keeps offsets into it
        self.info = info
        self.handle = handle

    def fetch(self) -> dict:
        info = self.info
        out = {k: np.empty(getattr(info, n), dtype=t) for k, (t, n) in _DOT_FIELDS.items()}
        out["slow"] = np.empty(2 * info.n_slow, dtype=np.int64)
        h = HsDotHost(**{k: v.ctypes.data if v.size else None for k, v in out.items()})
        check(_need(_dot_fetch, "hs_dot_fetch")(self.handle, ctypes.byref(h), stream_ptr()))
        return out

    def csr(self):
        """(root index, out_ptr, out_dst, ids, w_cpu, w_gpu, w_xfer, bytes) on the device."""
        n, m = ctypes.c_int64(), ctypes.c_int64()
        check(_need(_dot_csr_size, "hs_dot_csr_size")(self.handle, ctypes.byref(n),
                                                      ctypes.byref(m), stream_ptr()))
        n, m = n.value, m.value
        dev = self.text_dev.device
        e = lambda k, t: torch.empty(max(k, 1), dtype=t, device=dev)  # noqa: E731
        out_ptr, ids = e(n + 1, torch.int64), e(n, torch.int64)
        w_cpu, w_gpu = e(n, torch.float64), e(n, torch.float64)
        out_dst, w_xfer, nbytes = e(m, torch.int32), e(m, torch.float64), e(m, torch.int64)
        root = ctypes.c_int32()
        check(_need(_dot_csr, "hs_dot_csr")(self.handle, ptr(out_ptr), ptr(out_dst), ptr(ids),
                                            ptr(w_cpu), ptr(w_gpu), ptr(w_xfer), ptr(nbytes),
                                            ctypes.byref(root), stream_ptr()))
        return (root.value, out_ptr[:n + 1], out_dst[:m], ids[:n], w_cpu[:n], w_gpu[:n],
                w_xfer[:m], nbytes[:m])

    def close(self) -> None:
        if self.handle:
            _dot_release(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def dot_parse(data: bytes, device=None) -> Tuple[HsDotInfo, Optional[DotHandle]]:
    """Parse DOT bytes on the device (hs_dot_parse): (info, handle or None)."""
    dev = device or torch.device("cuda", torch.cuda.current_device())
    text = torch.empty(max(len(data), 1), dtype=torch.uint8, device=dev)
    if data:
        with warnings.catch_warnings():  # read-only view of the bytes: never written
            warnings.simplefilter("ignore", UserWarning)
            host = torch.frombuffer(data, dtype=torch.uint8)
        text[:len(data)].copy_(host)
    return dot_parse_device(text, len(data))


def dot_parse_device(text: torch.Tensor, nbytes: int) -> Tuple[HsDotInfo, Optional[DotHandle]]:
    """hs_dot_parse on DOT bytes already in device memory (uint8 tensor)."""
    info = HsDotInfo()
    handle = ctypes.c_void_p()
    check(_need(_dot_parse, "hs_dot_parse")(ptr(text), int(nbytes), ctypes.byref(info),
                                            ctypes.byref(handle), stream_ptr()))
    return info, (DotHandle(text, info, handle.value) if handle.value else None)


def dot_py_float(data: bytes) -> Tuple[int, float]:
    """(status, value) of the device's float() restated on the host (tests)."""
    out = ctypes.c_double()
    st = _need(_dot_py_float, "hs_dot_py_float")(data, len(data), ctypes.byref(out))
    return int(st), out.value
