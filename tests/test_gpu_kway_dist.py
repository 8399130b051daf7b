"""Sharded k-way partition (config 4 at 2/4/8 GPUs) on one GPU.

`loopback` runs P ranks as host threads on separate streams of one device:
every cross-rank exchange (replicated part / state / fine->coarse map stores,
the in-kernel all-reduce over the arenas) is the multi-GPU code path. The
two-process test maps the arenas with CUDA IPC like one process per GPU.
Checks: every rank returns the same partition; the reported cut equals an
independent recount; balance within tol; determinism; the sharded result is
a pure function of (graph, ranges, seed); quality close to one GPU.
"""
import numpy as np
import pytest
import torch

from paper_1502_07451_b200 import kway

pytestmark = pytest.mark.gpu


def _recount(csr, part):
    """Cut (each undirected edge once) and part loads from the full symmetrised graph."""
    ug = kway.symmetrize(csr)
    deg = (ug.xadj[1:] - ug.xadj[:-1])
    src = torch.repeat_interleave(torch.arange(ug.n, device=deg.device), deg)
    p = part.long()
    cut2 = (ug.adjwgt.long() * (p[src] != p[ug.adjncy.long()]).long()).sum().item()
    return cut2 // 2, ug


def _check(csr, res_list, k, tol=0.03):
    parts = [r.part for r in res_list]
    for p in parts[1:]:
        assert torch.equal(p, parts[0]), "ranks disagree on the partition"
    cuts = {r.cut for r in res_list}
    assert len(cuts) == 1
    cut, ug = _recount(csr, parts[0])
    assert cut == res_list[0].cut
    p = parts[0].long()
    assert p.min().item() >= 0 and p.max().item() < k
    loads = torch.zeros(k, dtype=torch.int64, device=p.device).index_add_(0, p, ug.vwgt.long())
    frac = (loads.double() / loads.sum().double()).cpu().numpy()
    assert np.abs(frac - 1.0 / k).max() <= tol + 1e-12
    assert all(r.feasible for r in res_list)
    return cut


@pytest.mark.parametrize("nranks", [2, 4])
def test_loopback_sharded_partition(nranks):
    csr = kway.layered_dag(200_000, 2_000_000, seed=3)
    k = 8
    res = kway.partition_kway_loopback(csr, nranks, k, seed=1)
    cut = _check(csr, res, k)
    single = kway.partition_kway(csr, k, seed=1)
    # local matching only: a little coarser coarsening, the cut stays close
    assert cut <= 1.10 * single.cut, (cut, single.cut)
    again = kway.partition_kway_loopback(csr, nranks, k, seed=1)
    assert torch.equal(again[0].part, res[0].part)


def test_loopback_small_and_uneven():
    """Small graph, more parts than ranks, non-uniform targets."""
    csr = kway.layered_dag(3_000, 30_000, seed=5)
    tp = [0.1, 0.2, 0.3, 0.4]
    res = kway.partition_kway_loopback(csr, 3, 4, tpwgts=tp, tol=0.05, seed=2)
    parts = [r.part for r in res]
    for p in parts[1:]:
        assert torch.equal(p, parts[0])
    cut, ug = _recount(csr, parts[0])
    assert cut == res[0].cut
    loads = torch.zeros(4, dtype=torch.int64, device=ug.vwgt.device).index_add_(
        0, parts[0].long(), ug.vwgt.long())
    frac = (loads.double() / loads.sum().double()).cpu().numpy()
    assert np.abs(frac - np.array(tp)).max() <= 0.05 + 1e-12


def test_one_rank_group_is_the_single_gpu_path():
    csr = kway.layered_dag(20_000, 200_000, seed=7)
    a = kway.partition_kway_loopback(csr, 1, 8, seed=0)[0]
    b = kway.partition_kway(csr, 8, seed=0)
    assert torch.equal(a.part, b.part) and a.cut == b.cut


def test_arena_too_small_is_an_error():
    from paper_1502_07451_b200 import _native
    csr = kway.layered_dag(5_000, 50_000, seed=1)
    ranges = kway.shard_ranges(csr, 2)
    ug = kway.symmetrize_range(csr, *ranges[0])
    g = kway.PartitionGroup(csr.n - 1, 2)
    d = g.dist(0)
    d.arena_bytes = 1024
    part = torch.empty(csr.n - 1, dtype=torch.int32, device="cuda")
    import ctypes
    with pytest.raises(_native.NativeError, match="arena"):
        tp = (ctypes.c_double * 2)(0.5, 0.5)
        stats = (ctypes.c_int64 * 8)()
        _native.check(_native._partition_kway_dist(
            ctypes.byref(ug.struct()), ranges[0][0], csr.n - 1, ctypes.byref(d), 2, tp, 0.03,
            ctypes.c_uint64(0), part.data_ptr(), stats, _native.stream_ptr()))


def _ipc_worker(rank, world, port, out):
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    torch.cuda.set_device(0)
    csr = kway.layered_dag(100_000, 1_000_000, seed=11)
    ranges = kway.shard_ranges(csr, world)
    ew = kway.integer_weights(csr.w_xfer)
    ug = kway.symmetrize_range(csr, *ranges[rank], ew, kway.integer_weights(csr.w_gpu),
                               kway.in_order(csr, ew))
    g = kway.PartitionGroup(csr.n - 1, world, mode="ipc", rank=rank)
    torch.cuda.synchronize()
    dist.barrier()
    r = kway.partition_kway_shard(ug, ranges[rank][0], csr.n - 1, g, rank, 8, seed=4)
    torch.cuda.synchronize()
    h = torch.tensor([r.cut, int(r.part.long().sum().item()),
                      int((r.part.long() * torch.arange(csr.n - 1, device="cuda")).sum().item())],
                     dtype=torch.int64)
    res = [torch.zeros(3, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(res, h)
    if rank == 0:
        out.put([x.tolist() for x in res])
    dist.barrier()
    dist.destroy_process_group()


def test_two_process_ipc_matches_loopback():
    import socket
    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    procs = [ctx.Process(target=_ipc_worker, args=(r, 2, port, out)) for r in range(2)]
    for p in procs:
        p.start()
    res = out.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
    assert all(p.exitcode == 0 for p in procs)
    assert res[0] == res[1]
    csr = kway.layered_dag(100_000, 1_000_000, seed=11)
    lb = kway.partition_kway_loopback(csr, 2, 8, seed=4)[0]
    p = lb.part.long()
    assert res[0] == [lb.cut, int(p.sum().item()),
                      int((p * torch.arange(csr.n - 1, device="cuda")).sum().item())]


@pytest.mark.parametrize("nranks,uniform", [(2, True), (3, False)])
def test_row_slices_give_the_same_shards_and_partition(nranks, uniform):
    """e2e at N > 1 ships each rank only its rows (kway.row_slice): K1 over a
    slice writes the rank's rows of the whole graph bit for bit, so the
    sharded partition is the same."""
    csr = kway.layered_dag(100_000, 1_000_000, seed=11)
    if uniform:
        ew = kway.integer_weights(csr.w_xfer)
    else:
        gen_ = torch.Generator(device="cpu").manual_seed(5)
        ew = torch.randint(1, 101, (csr.m,), generator=gen_, dtype=torch.int32).to(csr.device)
    ew_in = kway.in_order(csr, ew)
    nw = kway.integer_weights(csr.w_gpu)
    h = [a.cpu().numpy() for a in (csr.out_ptr, csr.out_dst, csr.in_ptr, csr.in_src, ew, ew_in, nw)]
    w0 = kway._uniform_weight(ew)  # the decision over all ranks' weights
    ranges = kway.shard_ranges(csr, nranks)
    full = [kway.symmetrize_range(csr, a, b, ew, nw, ew_in) for a, b in ranges]
    sliced = []
    for (a, b), f in zip(ranges, full):
        sl = kway.row_slice(*h, a, b)
        dev = {k: torch.from_numpy(sl[k]).to(csr.device) for k in kway.ROW_SLICE_KEYS}
        ug = kway.symmetrize_slice({**sl, **dev}, unit_weight=w0)
        assert torch.equal(ug.xadj, f.xadj) and torch.equal(ug.adjncy, f.adjncy)
        assert torch.equal(ug.vwgt, f.vwgt) and ug.unit_weight == f.unit_weight
        assert (ug._adjwgt is None) == (f._adjwgt is None)
        if f._adjwgt is not None:
            assert torch.equal(ug._adjwgt, f._adjwgt)
        sliced.append(ug)
    a = kway.partition_kway_loopback(csr, nranks, 8, seed=3, shards=full)[0]
    b = kway.partition_kway_loopback(csr, nranks, 8, seed=3, shards=sliced)[0]
    assert a.cut == b.cut and torch.equal(a.part, b.part)
