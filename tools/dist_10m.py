"""Loopback sharded partition of the config-4 DAG (10M/100M) at P ranks vs one GPU: cut, balance."""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1502_07451_b200 import kway

P = int(sys.argv[1]) if len(sys.argv) > 1 else 8
csr = kway.layered_dag(10_000_000, 100_000_000, seed=0)
single = kway.partition_kway(csr, 8, tol=0.03, seed=0)
torch.cuda.synchronize()
t = time.perf_counter()
res = kway.partition_kway_loopback(csr, P, 8, tol=0.03, seed=0)
torch.cuda.synchronize()
dt = time.perf_counter() - t
same = all(torch.equal(r.part, res[0].part) for r in res)
print(f"P={P} cut {res[0].cut} vs single {single.cut} ratio {res[0].cut / single.cut:.4f} "
      f"feasible {res[0].feasible} maxdev {res[0].max_deviation:.4f} levels {res[0].levels} "
      f"coarsest {res[0].coarsest} ranks_agree {same} loopback_wall_s {dt:.2f}")
