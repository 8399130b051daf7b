"""A/B timing of K1 symmetrize + the partition between two builds (argv[1] = package root)."""
import os
import sys
root = sys.argv[1]
sys.path.insert(0, root)
import torch
from paper_1502_07451_b200 import kway, _native
print("lib", _native.LIB_PATH)
csr = kway.layered_dag(10_000_000, 100_000_000, seed=0)
ew = kway.integer_weights(csr.w_xfer)
ew_in = kway.in_order(csr, ew)
nw = kway.integer_weights(csr.w_gpu)
for name, fn in (("symmetrize", lambda: kway.symmetrize(csr, ew, nw, ew_in)),
                 ("sym+partition", lambda: kway.partition_kway(kway.symmetrize(csr, ew, nw, ew_in), 8))):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        r = fn()
    b.record()
    torch.cuda.synchronize()
    print(name, a.elapsed_time(b) / 10, "ms")
