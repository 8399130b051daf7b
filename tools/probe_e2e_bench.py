"""The bench's e2e step in isolation, with and without the side-stream weight copy."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1502_07451_b200 import kway
from paper_1502_07451_b200.csr import DagCSR
dev = torch.device("cuda")
csr = kway.layered_dag(10_000_000, 100_000_000, 0)
ew, nw = kway.integer_weights(csr.w_xfer), kway.integer_weights(csr.w_gpu)
host = {k: getattr(csr, k).cpu().pin_memory() for k in ("out_ptr", "out_dst")}
hew, hnw = ew.cpu().pin_memory(), nw.cpu().pin_memory()
part_host = torch.empty(csr.n - 1, dtype=torch.int32).pin_memory()
side = torch.cuda.Stream(device=dev)


def step(use_side):
    main = torch.cuda.current_stream()
    d = {k: v.to(dev, non_blocking=True) for k, v in host.items()}
    if use_side:
        copied = torch.cuda.Event()
        copied.record(main)
        side.wait_event(copied)
        with torch.cuda.stream(side):
            ew_d = hew.to(dev, non_blocking=True)
            nw_d = hnw.to(dev, non_blocking=True)
    else:
        ew_d, nw_d = hew.to(dev, non_blocking=True), hnw.to(dev, non_blocking=True)
    g = DagCSR.from_out_csr(csr.root, d["out_ptr"], d["out_dst"])
    if use_side:
        main.wait_stream(side)
        ew_d.record_stream(main)
        nw_d.record_stream(main)
    r = kway.partition_kway(kway.symmetrize(g, ew_d, nw_d, None), 8, tol=0.03, seed=0)
    part_host.copy_(r.part, non_blocking=True)


for use_side in (False, True, False, True):
    step(use_side)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    a.record()
    for _ in range(3):
        step(use_side)
    b.record()
    torch.cuda.synchronize()
    print(f"side={use_side}: {a.elapsed_time(b) / 3:.2f} ms/step (wall {(time.perf_counter() - t0) / 3 * 1e3:.2f})",
          flush=True)
