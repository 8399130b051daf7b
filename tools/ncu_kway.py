"""One 10M-task partition for ncu captures (HS_NCU_LEVEL0 window; plain -k filters for K1/transpose)."""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1502_07451_b200 import kway

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
csr = kway.layered_dag(n, 10 * n, 0)
from paper_1502_07451_b200.csr import DagCSR
DagCSR.from_out_csr(csr.root, csr.out_ptr, csr.out_dst)  # hs_dag_transpose (e2e path)
ew = kway.integer_weights(csr.w_xfer)
ug = kway.symmetrize(csr, ew, kway.integer_weights(csr.w_gpu), kway.in_order(csr, ew))
r = kway.partition_kway(ug, 8, tol=0.03, seed=0)
torch.cuda.synchronize()
print("cut", r.cut, "levels", r.levels, "passes", r.refine_passes)
