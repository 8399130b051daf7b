"""Per-call timing of repeated 10M partitions (events + wall) to expose variance."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1502_07451_b200 import kway
csr = kway.layered_dag(10_000_000, 100_000_000, 0)
ew, nw = kway.integer_weights(csr.w_xfer), kway.integer_weights(csr.w_gpu)
ewi = kway.in_order(csr, ew)
torch.cuda.synchronize()
for i in range(30):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter(); a.record()
    ug = kway.symmetrize(csr, ew, nw, ewi)
    r = kway.partition_kway(ug, 8, seed=0)
    b.record(); torch.cuda.synchronize(); t1 = time.perf_counter()
    print(f"call {i}: events {a.elapsed_time(b):7.2f} ms  wall {1e3*(t1-t0):7.2f} ms  "
          f"mem_reserved {torch.cuda.memory_reserved()/1e9:.1f} GB", flush=True)
