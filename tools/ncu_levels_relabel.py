"""One K7 frontier launch (levels_kernel) on the config-4 DAG under a random
numbering (for ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1502_07451_b200 import kway
csr = kway.layered_dag(10_000_000, 100_000_000, 0)
rel, _ = kway.relabeled_dag(csr, seed=1)
del csr
torch.cuda.synchronize()
lv, fin, cp, nl = kway.levels(rel)
print("levels", nl, "cp", cp)
