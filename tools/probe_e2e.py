"""Phase times of the bench's e2e step (10M/100M), serialised with events."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1502_07451_b200 import kway
from paper_1502_07451_b200.csr import DagCSR
dev = torch.device("cuda")
csr = kway.layered_dag(10_000_000, 100_000_000, 0)
ew, nw = kway.integer_weights(csr.w_xfer), kway.integer_weights(csr.w_gpu)
h = {k: getattr(csr, k).cpu().pin_memory() for k in ("out_ptr", "out_dst")}
hew, hnw = ew.cpu().pin_memory(), nw.cpu().pin_memory()
ph = torch.empty(csr.n - 1, dtype=torch.int32).pin_memory()
torch.cuda.synchronize()
for it in range(3):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(7)]
    ev[0].record()
    d = {k: v.to(dev, non_blocking=True) for k, v in h.items()}
    ev[1].record()
    g = DagCSR.from_out_csr(csr.root, d["out_ptr"], d["out_dst"])
    ev[2].record()
    ewd, nwd = hew.to(dev, non_blocking=True), hnw.to(dev, non_blocking=True)
    ev[3].record()
    ug = kway.symmetrize(g, ewd, nwd)
    ev[4].record()
    r = kway.partition_kway(ug, 8, tol=0.03, seed=0)
    ev[5].record()
    ph.copy_(r.part, non_blocking=True)
    ev[6].record()
    torch.cuda.synchronize()
    names = ["h2d csr", "transpose", "h2d weights", "symmetrize", "partition", "d2h part"]
    print(it, " ".join(f"{n}={ev[i].elapsed_time(ev[i + 1]):.2f}" for i, n in enumerate(names)),
          f"total={ev[0].elapsed_time(ev[6]):.2f}", flush=True)
