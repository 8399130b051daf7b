"""compare() with the iterations split over ranks (batched DES
shards by simulation index, no exchange on the data path): two processes on
this GPU, gloo for the gather, each generating and simulating its half of the
seeds on the device; both return the rows one device returns, bit for bit."""
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

POLICIES = ["eager", "dmda", "gp"]


def _worker(rank, world, port, iterations, q):
    import torch
    from paper_1502_07451_b200 import gen, sim
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    fac = gen.RandomDagFactory(38, 75, "MA", 1024)
    rows = sim.compare_distributed(POLICIES, fac, sim.MachineModel(3, 1), iterations, seed=7)
    q.put((rank, [vars(r) for r in rows]))
    dist.barrier()
    dist.destroy_process_group()


def test_two_ranks_equal_one_device():
    from paper_1502_07451_b200 import gen, sim
    iterations = 515
    fac = gen.RandomDagFactory(38, 75, "MA", 1024)
    one = [vars(r) for r in sim.compare(POLICIES, fac, sim.MachineModel(3, 1), iterations, seed=7)]
    assert [vars(r) for r in sim.compare_distributed(POLICIES, fac, sim.MachineModel(3, 1),
                                                     iterations, seed=7)] == one
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, iterations, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=120)
    assert all(p.exitcode == 0 for p in procs)
    for _, rows in got:
        assert rows == one
