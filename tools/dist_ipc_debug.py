"""Two processes on one GPU, arenas CUDA-IPC mapped: the one-process-per-GPU path."""
import os
import socket
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.multiprocessing as mp


def worker(rank, world, port, n):
    import torch.distributed as dist
    from paper_1502_07451_b200 import kway
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    torch.cuda.set_device(0)
    csr = kway.layered_dag(n, 10 * n, seed=11)
    ranges = kway.shard_ranges(csr, world)
    if os.environ.get("DBG_EWIN"):
        ew = kway.integer_weights(csr.w_xfer)
        ug = kway.symmetrize_range(csr, *ranges[rank], ew, kway.integer_weights(csr.w_gpu),
                                   kway.in_order(csr, ew))
    else:
        ug = kway.symmetrize_range(csr, *ranges[rank])
    torch.cuda.synchronize()
    print(rank, "symmetrized", ranges[rank], flush=True)
    g = kway.PartitionGroup(csr.n - 1, world, mode="ipc", rank=rank)
    torch.cuda.synchronize()
    print(rank, "group", [hex(p) for p in g.ptrs], flush=True)
    dist.barrier()
    r = kway.partition_kway_shard(ug, ranges[rank][0], csr.n - 1, g, rank, 8, seed=4)
    print(rank, "returned cut", r.cut, flush=True)
    torch.cuda.synchronize()
    print(rank, "synced", r.part[:8].tolist(), flush=True)
    h = [r.cut, int(r.part.long().sum().item()),
         int((r.part.long() * torch.arange(csr.n - 1, device="cuda")).sum().item())]
    print(rank, "hash", h, flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 3000
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mp.spawn(worker, args=(2, port, n), nprocs=2)
