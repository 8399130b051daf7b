"""One 2-way ordered evaluate (K2 mode 0) on the config-2 DAG (for ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1502_07451_b200 import _native, kway
csr = kway.layered_dag(100_000, 1_000_000, 0)
nk = csr.n - 1
two = torch.ones((1, nk), dtype=torch.int8, device=csr.device)
two[0, :nk // 5] = 0
c, cw, t = _native.evaluate2(csr, two, 1, 0)
torch.cuda.synchronize()
print(float(c[0]), float(cw[0]))
