"""N>1 host logic on CPU with torch.distributed gloo, world_size 2.

The GPU data path cannot run here; what is shared by every rank and must agree
is host logic: the DAG task table, the owner maps (2D block-cyclic and the
partition-based one's contract), the expected transfer counts that the
executors' copy counters are checked against, and bench.py's max/sum-over-
ranks reductions.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1502_07451_b200.gen import cholesky_tasks

KIND = {"POTRF": 0, "TRSM": 1, "SYRK": 2, "GEMM": 3}


def _owner_cyclic(tasks, nranks):
    pr = int(np.floor(np.sqrt(nranks)))
    while nranks % pr:
        pr -= 1
    pc = nranks // pr
    out = []
    for kind, (i, j, k) in tasks:
        kd = KIND[kind]
        r = k if kd == 0 else i
        c = j if kd == 3 else (i if kd == 2 else k)
        out.append((r % pr) * pc + (c % pc))
    return np.array(out, dtype=np.int8)


def _transfers(deps, owner):
    d = np.array(deps) - 1
    po, co = owner[d[:, 0]], owner[d[:, 1]]
    cross = po != co
    return len(set(zip(d[cross, 0].tolist(), co[cross].tolist())))


def _worker(rank, world, port, T, q):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    tasks, deps = cholesky_tasks(T)
    owner = _owner_cyclic(tasks, world)
    # every rank derives the same owner map and transfer count
    mine = torch.tensor([float(owner.astype(np.int64).sum()), float(_transfers(deps, owner))])
    allv = [torch.zeros(2) for _ in range(world)]
    dist.all_gather(allv, mine)
    # work owned per rank (flops units b^3/3: POTRF 1, TRSM 3, SYRK 3, GEMM 6)
    w = np.array([{0: 1, 1: 3, 2: 3, 3: 6}[KIND[k]] for k, _ in tasks])
    load = torch.tensor([float(w[owner == rank].sum())])
    loads = [torch.zeros(1) for _ in range(world)]
    dist.all_gather(loads, load)
    # bench.py's max-over-ranks of a per-rank time
    t = torch.tensor([1.0 + rank])
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        q.put({"agree": all(torch.equal(allv[0], x) for x in allv),
               "transfers": float(allv[0][1]), "loads": [float(x) for x in loads],
               "total": float(w.sum()), "max_t": float(t)})
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("T", [8, 16])
def test_two_rank_owner_maps_agree_and_balance(T):
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, T, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
    assert all(p.exitcode == 0 for p in procs)
    assert res["agree"]
    assert res["max_t"] == 2.0
    assert sum(res["loads"]) == res["total"]
    assert max(res["loads"]) / (res["total"] / 2) < 1.2  # cyclic map balances work
    tasks, deps = cholesky_tasks(T)
    assert res["transfers"] == _transfers(deps, _owner_cyclic(tasks, 2)) > 0


# ---- sharded partition: every rank must derive the same vertex ranges -----

def _degrees(n, seed):
    rng = np.random.default_rng(seed)
    # layered-DAG-like skew: early kernels have many successors
    return (10 + rng.poisson(20.0 * (1.0 - np.arange(n) / n))).astype(np.int64)


def _range_worker(rank, world, port, n, q):
    from paper_1502_07451_b200.kway import split_bounds
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    cs = np.cumsum(_degrees(n, seed=5))
    b = split_bounds(cs, world)
    mine = torch.tensor([x for ab in b for x in ab], dtype=torch.int64)
    allb = [torch.zeros_like(mine) for _ in range(world)]
    dist.all_gather(allb, mine)
    # each rank's share of adjacency entries (what its kernels will scan)
    a, e = b[rank]
    share = torch.tensor([int(cs[e - 1] - (cs[a - 1] if a else 0))], dtype=torch.int64)
    shares = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(shares, share)
    if rank == 0:
        q.put({"agree": all(torch.equal(allb[0], x) for x in allb), "bounds": b,
               "shares": [int(s) for s in shares], "total": int(cs[-1])})
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_shard_ranges_agree_and_balance():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_range_worker, args=(r, 2, port, 50_000, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
    assert all(p.exitcode == 0 for p in procs)
    assert res["agree"]
    b = res["bounds"]
    assert b[0][0] == 0 and b[-1][1] == 50_000 and b[0][1] == b[1][0]
    assert sum(res["shares"]) == res["total"]
    assert max(res["shares"]) <= res["total"] / 2 * 1.01  # balanced by entries, not by count


def test_split_bounds_edge_cases():
    from paper_1502_07451_b200.kway import split_bounds
    cs = np.cumsum(np.ones(10, dtype=np.int64))
    assert split_bounds(cs, 1) == [(0, 10)]
    assert split_bounds(cs, 10) == [(i, i + 1) for i in range(10)]
    assert split_bounds(cs, 2) == [(0, 5), (5, 10)]
    # one huge vertex: every rank still gets >= 1 vertex
    cs = np.cumsum(np.array([1000, 1, 1, 1], dtype=np.int64))
    b = split_bounds(cs, 4)
    assert [e - a for a, e in b] == [1, 1, 1, 1]
    with pytest.raises(ValueError):
        split_bounds(cs, 5)


def _compare_arrays(iterations):
    rng = np.random.default_rng(9)
    return {name: (rng.uniform(10, 40, iterations), rng.integers(0, 30, iterations).astype(float),
                   rng.integers(0, 10 ** 9, iterations).astype(float))
            for name in ("eager", "dmda", "gp")}


def _compare_worker(rank, world, port, iterations, q):
    """sim.compare_distributed's host half: each rank holds the per-iteration
    results of its iteration_split share; gather_rows must give every rank the
    rows of all iterations in seed order."""
    from paper_1502_07451_b200.sim import gather_rows, iteration_split
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    full = _compare_arrays(iterations)
    mine = iteration_split(iterations, world, rank)
    local = {k: tuple(a[mine.start:mine.stop] for a in v) for k, v in full.items()}
    rows = gather_rows(["eager", "dmda", "gp"], local)
    q.put((rank, [vars(r) for r in rows], (mine.start, mine.stop)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("iterations", [4096, 1001, 1])
def test_two_rank_compare_rows_match_one_device(iterations):
    from paper_1502_07451_b200.sim import _row
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_compare_worker, args=(r, 2, port, iterations, q))
             for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
    assert all(p.exitcode == 0 for p in procs)
    full = _compare_arrays(iterations)
    want = [vars(_row(k, *full[k])) for k in ("eager", "dmda", "gp")]
    spans = sorted(g[2] for g in got)
    assert spans[0][0] == 0 and spans[-1][1] == iterations and spans[0][1] == spans[1][0]
    for _, rows, _ in got:
        assert rows == want  # bit-identical on every rank


def _small_dag(n, m, seed):
    """Random DAG with root 0 feeding every node without a predecessor: the
    host CSR arrays (out sorted by (src, dst), in ascending by source)."""
    rng = np.random.default_rng(seed)
    src = rng.integers(1, n - 1, m)
    dst = np.minimum(n - 1, src + 1 + rng.integers(0, 50, m))
    e = np.unique(np.stack([src, dst], 1), axis=0)
    has_pred = np.zeros(n, bool)
    has_pred[e[:, 1]] = True
    roots = np.nonzero(~has_pred[1:])[0] + 1
    e = np.concatenate([np.stack([np.zeros_like(roots), roots], 1), e])
    e = e[np.lexsort((e[:, 1], e[:, 0]))]
    out_ptr = np.zeros(n + 1, np.int64)
    np.add.at(out_ptr, e[:, 0] + 1, 1)
    out_ptr = np.cumsum(out_ptr)
    ew = rng.integers(1, 100, len(e)).astype(np.int32)
    order = np.lexsort((e[:, 0], e[:, 1]))
    in_ptr = np.zeros(n + 1, np.int64)
    np.add.at(in_ptr, e[:, 1] + 1, 1)
    in_ptr = np.cumsum(in_ptr)
    nw = rng.integers(1, 100, n).astype(np.int32)
    return (out_ptr, e[:, 1].astype(np.int32), in_ptr, e[order, 0].astype(np.int32), ew,
            ew[order], nw)


def _rows(out_ptr, out_dst, in_ptr, in_src, ew, ew_in, nw, v0, v1):
    """K1's rows for nodes [v0, v1) of a DAG with root 0: in-list (root dropped)
    then out-list, kernel ids u - 1, with weights (the kernel's definition)."""
    rows = []
    for v in range(v0, v1):
        a, b = in_ptr[v], in_ptr[v + 1]
        ins = [(int(in_src[j]) - 1, int(ew_in[j])) for j in range(a, b) if in_src[j] != 0]
        outs = [(int(out_dst[j]) - 1, int(ew[j])) for j in range(out_ptr[v], out_ptr[v + 1])]
        rows.append((int(nw[v]), ins + outs))
    return rows


def _slice_worker(rank, world, port, q):
    from paper_1502_07451_b200.kway import row_slice, split_bounds
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    full = _small_dag(3000, 12000, 4)
    out_ptr, out_dst, in_ptr, in_src, ew, ew_in, nw = full
    n = len(out_ptr) - 1
    deg = (np.diff(in_ptr) + np.diff(out_ptr))[1:]
    kv0, kv1 = split_bounds(np.cumsum(deg), world)[rank]
    sl = row_slice(*full, kv0, kv1)
    # the rank's rows from its slice alone (local rows 1..nl, global neighbour ids)
    mine = _rows(sl["out_ptr"], sl["out_dst"], sl["in_ptr"], sl["in_src"], sl["ew"],
                 sl["ew_in"], sl["nw"], 1, kv1 - kv0 + 1)
    want = _rows(*full, kv0 + 1, kv1 + 1)
    sizes = torch.tensor([sum(len(r[1]) for r in mine), int(sl["nnz"]),
                          sum(int(sl[k].nbytes) for k in ("out_ptr", "out_dst", "in_ptr",
                                                            "in_src", "ew", "ew_in", "nw"))])
    alls = [torch.zeros(3, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(alls, sizes)
    full_nnz = sum(len(r[1]) for r in _rows(*full, 1, n))
    full_bytes = sum(int(a.nbytes) for a in full)
    q.put((rank, mine == want, [x.tolist() for x in alls], full_nnz, full_bytes))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_row_slices_carry_their_rows():
    """The e2e row-range split: each rank's row_slice alone
    yields exactly its K1 rows of the whole graph, the slices' entries add up
    to the graph's, and each rank ships a fraction of the whole DAG."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_slice_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
    assert all(p.exitcode == 0 for p in procs)
    for rank, same, alls, full_nnz, full_bytes in got:
        assert same
        assert all(a[0] == a[1] for a in alls)  # nnz predicted = entries built
        assert sum(a[0] for a in alls) == full_nnz
        assert all(a[2] < 0.75 * full_bytes for a in alls)
