"""One K7 launch on the 10M DAG (for ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1502_07451_b200 import kway
csr = kway.layered_dag(int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000,
                       int(sys.argv[2]) if len(sys.argv) > 2 else 100_000_000, 0)
torch.cuda.synchronize()
lv, fin, cp, nl = kway.levels(csr)
h = torch.bincount(lv.long()).cpu().tolist()
print("levels", nl, "sizes", h[:8], "...", h[-8:], "max", max(h))
