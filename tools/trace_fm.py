"""HS_KWAY_TRACE run of one partition (FM level counters on stderr)."""
import os, sys, time
sys.path.insert(0, sys.argv[1] if len(sys.argv) > 1 else ".")
import torch
from paper_1502_07451_b200 import kway
n = int(sys.argv[2]) if len(sys.argv) > 2 else 20_000
k = int(sys.argv[3]) if len(sys.argv) > 3 else 8
csr = kway.layered_dag(n, 10 * n, seed=1)
ug = kway.symmetrize(csr)
r = kway.partition_kway(ug, k, tol=0.03, seed=0)
torch.cuda.synchronize()
t0 = time.perf_counter()
r = kway.partition_kway(ug, k, tol=0.03, seed=0)
torch.cuda.synchronize()
print("cut", r.cut, "ms", (time.perf_counter() - t0) * 1e3, "levels", r.stats if hasattr(r, "stats") else "")
