"""One sym+partition of the 10M DAG with a given build (argv[1] = package root), for ncu A/B."""
import sys
sys.path.insert(0, sys.argv[1])
import torch
from paper_1502_07451_b200 import kway
csr = kway.layered_dag(10_000_000, 100_000_000, seed=0)
ew = kway.integer_weights(csr.w_xfer)
ew_in = kway.in_order(csr, ew)
nw = kway.integer_weights(csr.w_gpu)
for _ in range(2):
    r = kway.partition_kway(kway.symmetrize(csr, ew, nw, ew_in), 8)
torch.cuda.synchronize()
print("cut", r.cut)
