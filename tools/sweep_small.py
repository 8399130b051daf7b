"""Cut / time of k-way partitions of the smoke DAG (20k/200k), the tiled-Cholesky
DAG (T=32: 5,984 tasks; T=64: 45,760 tasks) under the current env knobs."""
import os, sys, time
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_1502_07451_b200 import kway, cholesky
from paper_1502_07451_b200.csr import DagCSR, HostDag


def chol_ug(T):
    table = cholesky.task_table(T)
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
    F = cholesky.TASK_FLOPS_B3
    w = np.array([0.0] + [float(F[k]) for k in kind])
    h = HostDag(ids, 0, src, dst, w, w, np.ones(len(src)), np.full(len(src), 8, dtype=np.int64))
    csr = DagCSR.from_host(h)
    ew = torch.ones(csr.m, dtype=torch.int32, device=csr.device)
    nw = torch.from_numpy(np.array([0] + [F[k] for k in kind], dtype=np.int32)).to(csr.device)
    return kway.symmetrize(csr, ew, nw, ew), n


def run(name, ug, k):
    kway.partition_kway(ug, k, tol=0.03, seed=0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        r = kway.partition_kway(ug, k, tol=0.03, seed=0)
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) / 3 * 1e3
    print(f"  {name:14s} k={k} cut {r.cut:12d} dev {r.max_deviation:.4f} {ms:8.2f} ms", flush=True)


csr = kway.layered_dag(20_000, 200_000, seed=1)
run("layered20k", kway.symmetrize(csr), 8)
for T in (32, 64):
    ug, n = chol_ug(T)
    for k in (2, 4, 8):
        run(f"chol{n}", ug, k)
