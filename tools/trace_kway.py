"""Phase trace (HS_KWAY_TRACE=1 -> stderr) of one 10M partition after two warm-up calls."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1502_07451_b200 import kway
csr = kway.layered_dag(10_000_000, 100_000_000, 0)
ew, nw = kway.integer_weights(csr.w_xfer), kway.integer_weights(csr.w_gpu)
ug = kway.symmetrize(csr, ew, nw, kway.in_order(csr, ew))
for _ in range(2):
    kway.partition_kway(ug, 8, seed=0)
torch.cuda.synchronize()
os.environ["HS_KWAY_TRACE"] = "1"
r = kway.partition_kway(ug, 8, seed=0)
torch.cuda.synchronize()
print("cut", r.cut, flush=True)
