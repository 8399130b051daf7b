"""Partitioned (multi-executor) Cholesky: the cross-partition protocol on one GPU.

`loopback` runs P executors concurrently on one device, each owning a DAG part;
cross-partition edges are real peer stores + inbox posts, exactly the
multi-GPU code path. Numerics vs LAPACK, copies == distinct transfer count.
"""
import numpy as np
import pytest
import torch

from paper_1502_07451_b200.cholesky import (PartitionedCholesky, owner_cyclic, owner_partition,
                                             spd_matrix, task_table, transfer_count)

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("nranks,mapper", [(2, "cyclic"), (4, "cyclic"), (2, "partition"),
                                           (4, "partition")])
def test_loopback_matches_lapack(nranks, mapper):
    n = 4096
    tb = task_table(n // 512)
    owner = owner_cyclic(tb, nranks) if mapper == "cyclic" else owner_partition(tb, nranks)
    assert owner.min() >= 0 and owner.max() < nranks
    pc = PartitionedCholesky(n, owner, nranks, mode="loopback")
    A = spd_matrix(n, seed=2)
    pc.load(A)
    pc.run()
    L = pc.result_loopback()
    ref = np.linalg.cholesky(A.cpu().numpy())
    err = np.abs(L.cpu().numpy() - ref).max() / np.abs(ref).max()
    assert err <= 1e-10, err
    # every cross-partition transfer was issued exactly once (K2 dedup rule)
    assert sum(pc.copies) == transfer_count(tb, owner) > 0


def _ipc_worker(rank, world, port, n, out):
    import os
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    torch.cuda.set_device(0)
    tb = task_table(n // 512)
    owner = owner_cyclic(tb, world)
    pc = PartitionedCholesky(n, owner, world, mode="ipc", rank=rank)
    A = spd_matrix(n, seed=4)
    pc.load(A)
    torch.cuda.synchronize()
    dist.barrier()
    pc.run()
    torch.cuda.synchronize()
    dist.barrier()
    # check the final tiles this rank owns against LAPACK
    from paper_1502_07451_b200.cholesky import _pack, TILE
    from paper_1502_07451_b200 import _native
    tmp = torch.zeros(n, n, dtype=torch.float64, device="cuda")
    _native.check(_pack(_native.ptr(tmp), n, TILE, pc.ranks[rank].tiles.data_ptr(), 0,
                        _native.stream_ptr()))
    ref = torch.from_numpy(np.linalg.cholesky(A.cpu().numpy()))
    err = 0.0
    for (i, j), q in pc.final_owner_of_tiles().items():
        if q == rank:
            sl = (slice(i * TILE, (i + 1) * TILE), slice(j * TILE, (j + 1) * TILE))
            err = max(err, (tmp[sl].cpu() - ref[sl]).abs().max().item())
    t = torch.tensor([err / ref.abs().max().item(), float(pc.copies[rank])], dtype=torch.float64)
    res = [torch.zeros(2, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(res, t)
    if rank == 0:
        out.put([r.tolist() for r in res])
    dist.barrier()
    dist.destroy_process_group()


def test_two_process_ipc_on_one_gpu():
    """Two processes (one per 'GPU'), peers mapped with CUDA IPC: the real multi-process path."""
    import socket
    import torch.multiprocessing as mp
    n = 4096
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    procs = [ctx.Process(target=_ipc_worker, args=(r, 2, port, n, out)) for r in range(2)]
    for p in procs:
        p.start()
    res = out.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
    assert all(p.exitcode == 0 for p in procs)
    errs = [r[0] for r in res]
    copies = sum(r[1] for r in res)
    assert max(errs) <= 1e-10, errs
    tb = task_table(n // 512)
    assert copies == transfer_count(tb, owner_cyclic(tb, 2))
