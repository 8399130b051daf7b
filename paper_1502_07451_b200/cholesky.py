"""Execution of the tiled-Cholesky task DAG on B200s (config 1 / config 3).

The reference schedules this DAG only in simulation (kernel_time from a
calibration table, sim.py:135-164); here the same DAG (``gen.cholesky_tasks``,
SURVEY App. D) is executed: one persistent sm_100a kernel per GPU pulls ready
tasks from device queues and runs POTRF/TRSM/SYRK/GEMM tiles on fp64 DMMA
(csrc/tile_cholesky.cu).

``TiledCholesky(n).factor(A)`` returns the lower Cholesky factor of an SPD
fp64 matrix resident on the device.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from . import _native
from .gen import cholesky_tasks

KIND_ID = {"POTRF": 0, "TRSM": 1, "SYRK": 2, "GEMM": 3}
TILE = 512

_P = ctypes.c_void_p
_pack = _native._proto("hs_chol_pack", _P, ctypes.c_int32, ctypes.c_int32, _P, ctypes.c_int32, _P)
_exec = _native._proto("hs_chol_execute_stats", _P, _P, ctypes.c_int32, ctypes.c_int32, _P, _P, _P,
                       _P, _P, _P, _P, ctypes.c_int32, _P, _P, _P)


@dataclass
class TaskTable:
    """Device arrays of the Cholesky task DAG (task t = id t+1 of the DAG)."""
    n_tasks: int
    kind: torch.Tensor      # int8
    ti: torch.Tensor        # int16
    tj: torch.Tensor
    tk: torch.Tensor
    succ_ptr: torch.Tensor  # int64 [n_tasks+1]
    succ: torch.Tensor      # int32
    indeg: torch.Tensor     # int32
    deps: np.ndarray        # host (producer, consumer) pairs, 0-based task indices


def task_table(tiles: int, device=None) -> TaskTable:
    dev = device or _native.device()
    tasks, deps = cholesky_tasks(tiles)
    n = len(tasks)
    kind = np.array([KIND_ID[k] for k, _ in tasks], dtype=np.int8)
    coords = np.array([key for _, key in tasks], dtype=np.int16)
    d = np.array(deps, dtype=np.int64).reshape(-1, 2) - 1  # 0-based
    order = np.lexsort((d[:, 1], d[:, 0]))
    d = d[order]
    succ_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(d[:, 0], minlength=n), out=succ_ptr[1:])
    indeg = np.bincount(d[:, 1], minlength=n).astype(np.int32)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    return TaskTable(n, t(kind), t(coords[:, 0]), t(coords[:, 1]), t(coords[:, 2]), t(succ_ptr),
                     t(d[:, 1].astype(np.int32)), t(indeg), d)


class TiledCholesky:
    """fp64 Cholesky of an n x n SPD matrix by the tiled task DAG, b = 512."""

    def __init__(self, n: int, device=None, grid_ctas: int = 0):
        if n % TILE:
            raise ValueError(f"n must be a multiple of {TILE}")
        self.n = n
        self.T = n // TILE
        self.device = device or _native.device()
        self.table = task_table(self.T, self.device)
        self.tiles = torch.empty(self.T * self.T * TILE * TILE, dtype=torch.float64,
                                 device=self.device)
        self.dinv = torch.empty(self.T * 4 * 128 * 128, dtype=torch.float64, device=self.device)
        self.grid_ctas = grid_ctas

    @property
    def flops(self) -> float:
        return self.n ** 3 / 3.0

    def load(self, A: torch.Tensor) -> None:
        """Row-major SPD matrix -> tile layout (lower tiles)."""
        assert A.dtype == torch.float64 and A.is_cuda and A.shape == (self.n, self.n)
        A = A.contiguous()
        _native.check(_pack(_native.ptr(A), self.n, TILE, _native.ptr(self.tiles), 1,
                            _native.stream_ptr()))

    def run(self, stats: Optional[torch.Tensor] = None) -> None:
        """Execute the DAG in place on the loaded tiles (optional u64[16] cycle stats)."""
        tb = self.table
        fail = ctypes.c_int32(0)
        _native.check(_exec(_native.ptr(self.tiles), _native.ptr(self.dinv), self.T, tb.n_tasks,
                            _native.ptr(tb.kind), _native.ptr(tb.ti), _native.ptr(tb.tj),
                            _native.ptr(tb.tk), _native.ptr(tb.succ_ptr), _native.ptr(tb.succ),
                            _native.ptr(tb.indeg), self.grid_ctas, ctypes.byref(fail),
                            _native.ptr(stats), _native.stream_ptr()))
        if fail.value:
            raise ValueError("matrix is not positive definite")

    def result(self, out: Optional[torch.Tensor] = None) -> torch.Tensor:
        """Lower factor L (row-major, strictly upper part zero)."""
        if out is None:
            out = torch.zeros(self.n, self.n, dtype=torch.float64, device=self.device)
        _native.check(_pack(_native.ptr(out), self.n, TILE, _native.ptr(self.tiles), 0,
                            _native.stream_ptr()))
        return out

    def factor(self, A: torch.Tensor) -> torch.Tensor:
        self.load(A)
        self.run()
        return self.result()


def spd_matrix(n: int, seed: int = 0, device=None) -> torch.Tensor:
    """SURVEY §8(d) input: A = R R^T + n I, R ~ N(0, 1) (fp64, on the device)."""
    dev = device or _native.device()
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    R = torch.randn(n, n, dtype=torch.float64, device=dev, generator=g)
    A = R @ R.T
    A.diagonal().add_(float(n))
    return A


# --------------------------------------------------------------------------
# Partitioned execution over several GPUs: rank r runs the
# tasks it owns; cross-partition edges become peer stores of the producer's
# output tile plus an inbox post (csrc/tile_cholesky.cu, hs_chol_execute_part).
# --------------------------------------------------------------------------

class HsCholPeers(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int32), ("nranks", ctypes.c_int32), ("owner", _P),
                ("tiles", _P * 8), ("dinv", _P * 8), ("inbox", _P * 8), ("ctl", _P * 8)]


_exec_part = _native._proto("hs_chol_execute_part", _P, _P, ctypes.c_int32, ctypes.c_int32, _P, _P,
                            _P, _P, _P, _P, _P, _P, ctypes.c_int32, _P, _P, _P, _P)
_ipc_handle = _native._proto("hs_ipc_handle", _P, ctypes.c_char_p)
_ipc_open = _native._proto("hs_ipc_open", ctypes.c_char_p, ctypes.POINTER(_P))
_ipc_close = _native._proto("hs_ipc_close", _P)
_ipc_alloc = _native._proto("hs_ipc_alloc", ctypes.c_int64, ctypes.POINTER(_P))
_ipc_free = _native._proto("hs_ipc_free", _P)
_memset = _native._proto("hs_memset_async", _P, ctypes.c_int32, ctypes.c_int64, _P)

TASK_FLOPS_B3 = {0: 1, 1: 3, 2: 3, 3: 6}  # task flops in units of b^3/3 (POTRF b^3/3 ... GEMM 2b^3)


def owner_cyclic(table: TaskTable, nranks: int) -> np.ndarray:
    """2D block-cyclic owner of each task's output tile (the ScaLAPACK baseline)."""
    pr = int(np.floor(np.sqrt(nranks)))
    while nranks % pr:
        pr -= 1
    pc = nranks // pr
    kind = table.kind.cpu().numpy()
    ti, tj, tk = (x.cpu().numpy().astype(np.int64) for x in (table.ti, table.tj, table.tk))
    r = np.where(kind == 0, tk, ti)
    c = np.where(kind == 3, tj, np.where(kind == 2, ti, tk))
    return ((r % pr) * pc + (c % pc)).astype(np.int8)


def owner_partition(table: TaskTable, nranks: int, tol: float = 0.03, seed: int = 0) -> np.ndarray:
    """Owner map from the multilevel k-way partitioner (the paper's policy, k = #GPUs).

    Vertex weight = task flops, edge weight = 1 tile; balance |w_p/W - 1/k| <= tol.
    """
    from .csr import DagCSR, HostDag
    from . import kway
    kind = table.kind.cpu().numpy()
    n = table.n_tasks
    d = table.deps
    ids = np.arange(n + 1, dtype=np.int64)
    has_pred = np.zeros(n, dtype=bool)
    has_pred[d[:, 1]] = True
    roots = np.nonzero(~has_pred)[0]
    src = np.concatenate([d[:, 0] + 1, np.zeros(len(roots), dtype=np.int64)])
    dst = np.concatenate([d[:, 1] + 1, roots + 1])
    o = np.lexsort((dst, src))
    src, dst = src[o].astype(np.int32), dst[o].astype(np.int32)
    w = np.array([0.0] + [float(TASK_FLOPS_B3[k]) for k in kind])
    h = HostDag(ids, 0, src, dst, w, w, np.ones(len(src)), np.full(len(src), TILE * TILE * 8,
                                                                    dtype=np.int64))
    csr = DagCSR.from_host(h)
    ew = torch.ones(csr.m, dtype=torch.int32, device=csr.device)
    nw = torch.from_numpy(np.array([0] + [TASK_FLOPS_B3[k] for k in kind], dtype=np.int32)
                          ).to(csr.device)
    ug = kway.symmetrize(csr, ew, nw, ew)
    res = kway.partition_kway(ug, nranks, tol=tol, seed=seed)
    return res.part.cpu().numpy().astype(np.int8)


def transfer_count(table: TaskTable, owner: np.ndarray) -> int:
    """Distinct (producer, remote consumer part) pairs = tile copies the executor issues."""
    d = table.deps
    po, co = owner[d[:, 0]], owner[d[:, 1]]
    cross = po != co
    return len(set(zip(d[cross, 0].tolist(), co[cross].tolist())))


class _Buf:
    """A whole cudaMalloc allocation (IPC-shareable), with a data_ptr() like a tensor."""

    def __init__(self, nbytes: int):
        p = _P()
        _native.check(_ipc_alloc(nbytes, ctypes.byref(p)))
        self.ptr, self.nbytes = p.value, nbytes

    def data_ptr(self) -> int:
        return self.ptr

    def fill_bytes(self, value: int) -> None:
        _native.check(_memset(self.ptr, value, self.nbytes, _native.stream_ptr()))

    def __del__(self):
        if getattr(self, "ptr", None):
            _ipc_free(self.ptr)
            self.ptr = None


class _Rank:
    def __init__(self, T, n_tasks, dev):
        self.tiles = _Buf(T * T * TILE * TILE * 8)
        self.dinv = _Buf(T * 4 * 128 * 128 * 8)
        self.inbox = _Buf(n_tasks * 8)
        self.ctl = _Buf(2 * 8)
        self.reset()

    def reset(self):
        self.inbox.fill_bytes(0xFF)  # -1
        self.ctl.fill_bytes(0)


class PartitionedCholesky:
    """Tiled Cholesky executed across `nranks` executors that own DAG parts.

    mode "loopback": all executors on this GPU (separate streams, SMs split) —
    exercises the exact cross-partition protocol on one device.
    mode "ipc": this process is rank `rank` of a torch.distributed group with one
    process per GPU; peers' buffers are mapped with CUDA IPC.
    """

    def __init__(self, n: int, owner: np.ndarray, nranks: int, mode: str = "loopback",
                 rank: int = 0, group=None, device=None):
        if n % TILE:
            raise ValueError(f"n must be a multiple of {TILE}")
        if not 1 <= nranks <= 8:
            raise ValueError("1..8 ranks")
        self.n, self.T, self.nranks, self.mode = n, n // TILE, nranks, mode
        self.device = device or _native.device()
        self.table = task_table(self.T, self.device)
        self.owner_host = np.asarray(owner, dtype=np.int8)
        self.owner = torch.from_numpy(self.owner_host).to(self.device)
        self.copies = [0] * nranks
        nt = self.table.n_tasks
        if mode == "loopback":
            self.ranks = [_Rank(self.T, nt, self.device) for _ in range(nranks)]
            self.peer_ptrs = [(r.tiles.data_ptr(), r.dinv.data_ptr(), r.inbox.data_ptr(),
                               r.ctl.data_ptr()) for r in self.ranks]
            self.my_ranks = list(range(nranks))
        elif mode == "ipc":
            import torch.distributed as dist
            self.rank = rank
            me = _Rank(self.T, nt, self.device)
            self.ranks = {rank: me}
            handles = []
            for t in (me.tiles, me.dinv, me.inbox, me.ctl):
                buf = ctypes.create_string_buffer(64)
                _native.check(_ipc_handle(t.data_ptr(), buf))
                handles.append(buf.raw)
            allh = [None] * nranks
            dist.all_gather_object(allh, handles, group=group)
            self.peer_ptrs, self._opened = [], []
            for q in range(nranks):
                if q == rank:
                    self.peer_ptrs.append((me.tiles.data_ptr(), me.dinv.data_ptr(),
                                           me.inbox.data_ptr(), me.ctl.data_ptr()))
                    continue
                ptrs = []
                for h in allh[q]:
                    p = _P()
                    _native.check(_ipc_open(h, ctypes.byref(p)))
                    ptrs.append(p.value)
                    self._opened.append(p.value)
                self.peer_ptrs.append(tuple(ptrs))
            self.my_ranks = [rank]
        else:
            raise ValueError(mode)

    def _peers(self, r: int) -> HsCholPeers:
        pe = HsCholPeers()
        pe.rank, pe.nranks, pe.owner = r, self.nranks, self.owner.data_ptr()
        for q, (t, d, i, c) in enumerate(self.peer_ptrs):
            pe.tiles[q], pe.dinv[q], pe.inbox[q], pe.ctl[q] = t, d, i, c
        return pe

    def load(self, A: torch.Tensor) -> None:
        """Every executor starts from the full input (tiles it never touches stay unused)."""
        A = A.contiguous()
        for r in self.my_ranks:
            rk = self.ranks[r]
            rk.reset()
            _native.check(_pack(_native.ptr(A), self.n, TILE, rk.tiles.data_ptr(), 1,
                                _native.stream_ptr()))

    def run(self, grid_ctas: int = 0) -> None:
        tb = self.table
        cur = torch.cuda.current_stream()
        if self.mode == "loopback":
            sms = torch.cuda.get_device_properties(self.device).multi_processor_count
            grid = grid_ctas or max(1, sms // self.nranks)
            streams = [torch.cuda.Stream(device=self.device) for _ in range(self.nranks)]
            for st in streams:
                st.wait_stream(cur)
            cps = torch.zeros(self.nranks, dtype=torch.int64, device=self.device)
            peers = [self._peers(r) for r in range(self.nranks)]
            for r in range(self.nranks):  # launch all before any sync: executors must co-run
                rk = self.ranks[r]
                _native.check(_exec_part(rk.tiles.data_ptr(), rk.dinv.data_ptr(), self.T,
                                         tb.n_tasks, _native.ptr(tb.kind), _native.ptr(tb.ti),
                                         _native.ptr(tb.tj), _native.ptr(tb.tk),
                                         _native.ptr(tb.succ_ptr), _native.ptr(tb.succ),
                                         _native.ptr(tb.indeg), ctypes.byref(peers[r]), grid, None,
                                         None, cps.data_ptr() + 8 * r, streams[r].cuda_stream))
            for st in streams:
                cur.wait_stream(st)
            torch.cuda.synchronize(self.device)
            self.copies = cps.cpu().tolist()
        else:
            rk = self.ranks[self.rank]
            peers = self._peers(self.rank)
            cp = torch.zeros(1, dtype=torch.int64, device=self.device)
            fail = ctypes.c_int32(0)
            _native.check(_exec_part(rk.tiles.data_ptr(), rk.dinv.data_ptr(), self.T,
                                     tb.n_tasks, _native.ptr(tb.kind), _native.ptr(tb.ti),
                                     _native.ptr(tb.tj), _native.ptr(tb.tk),
                                     _native.ptr(tb.succ_ptr), _native.ptr(tb.succ),
                                     _native.ptr(tb.indeg), ctypes.byref(peers), grid_ctas,
                                     ctypes.byref(fail), None, cp.data_ptr(),
                                     _native.stream_ptr()))
            self.copies[self.rank] = int(cp.item())
            if fail.value:
                raise ValueError("matrix is not positive definite")

    def final_owner_of_tiles(self) -> dict:
        """(i, j) -> rank holding the final L tile (owner of its POTRF/TRSM)."""
        kind = self.table.kind.cpu().numpy()
        ti, tk = self.table.ti.cpu().numpy(), self.table.tk.cpu().numpy()
        out = {}
        for t in np.nonzero(kind <= 1)[0]:
            i = int(tk[t]) if kind[t] == 0 else int(ti[t])
            out[(i, int(tk[t]))] = int(self.owner_host[t])
        return out

    def result_loopback(self) -> torch.Tensor:
        """Assemble L from the ranks' final tiles (loopback mode)."""
        L = torch.zeros(self.n, self.n, dtype=torch.float64, device=self.device)
        tmp = torch.zeros_like(L)
        for r in range(self.nranks):
            _native.check(_pack(_native.ptr(tmp), self.n, TILE, self.ranks[r].tiles.data_ptr(), 0,
                                _native.stream_ptr()))
            for (i, j), q in self.final_owner_of_tiles().items():
                if q == r:
                    sl = (slice(i * TILE, (i + 1) * TILE), slice(j * TILE, (j + 1) * TILE))
                    L[sl] = tmp[sl]
        return L
