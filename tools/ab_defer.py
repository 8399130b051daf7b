"""Deferred row updates A/B: the 10M partition with HS_KWAY_DEFER unset vs 0
(same process would cache the env; run twice). Prints cut, part hash, ms."""
import hashlib, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1502_07451_b200 import kway
csr = kway.layered_dag(10_000_000, 100_000_000, 0)
ew = kway.integer_weights(csr.w_xfer)
nw = kway.integer_weights(csr.w_gpu)
ug = kway.symmetrize(csr, ew, nw, kway.in_order(csr, ew))
for _ in range(3):
    r = kway.partition_kway(ug, 8, tol=0.03, seed=0)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(10):
    r = kway.partition_kway(ug, 8, tol=0.03, seed=0)
b.record()
torch.cuda.synchronize()
print("defer", os.environ.get("HS_KWAY_DEFER", "1"), "cut", r.cut,
      hashlib.sha1(r.part.cpu().numpy().tobytes()).hexdigest()[:12], "ms", a.elapsed_time(b) / 10)
