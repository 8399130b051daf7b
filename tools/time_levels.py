"""K7 timing on the 10M DAG: creation order (dataflow kernel) vs relabelled (frontier kernel)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1502_07451_b200 import kway
csr = kway.layered_dag(10_000_000, 100_000_000, 0)
def t(c, reps=5):
    kway.levels(c); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): r = kway.levels(c)
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps, r
ms, (lv, fin, cp, nl) = t(csr)
print("ordered  ms %.3f levels %d cp %r" % (ms, nl, cp))
rel, pi = kway.relabeled_dag(csr, 1)
del csr
ms2, (lv2, fin2, cp2, nl2) = t(rel)
print("relabeled ms %.3f levels %d cp %r equal %s" % (ms2, nl2, cp2, cp2 == cp and nl2 == nl))
