"""Small loopback sharded partition for debugging the exchange (HS_DIST_TRACE=1)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1502_07451_b200 import kway

n = int(sys.argv[1]) if len(sys.argv) > 1 else 3000
P = int(sys.argv[2]) if len(sys.argv) > 2 else 2
csr = kway.layered_dag(n, 10 * n, seed=3)
res = kway.partition_kway_loopback(csr, P, 8, seed=1)
torch.cuda.synchronize()
print("cuts", [r.cut for r in res], "feasible", [r.feasible for r in res],
      "same", all(torch.equal(r.part, res[0].part) for r in res))
print("single", kway.partition_kway(csr, 8, seed=1).cut)
