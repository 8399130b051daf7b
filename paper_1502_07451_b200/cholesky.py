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
