"""Small k-way partitions (coarsening + CTA FM + starts) for compute-sanitizer runs."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import torch
from paper_1502_07451_b200 import kway
import _kway_cases as KC
dev = torch.device("cuda")
c = KC.cases()[sys.argv[1] if len(sys.argv) > 1 else "L200"]()
xadj, adj, w, vw = KC.csr(c)
t = lambda a: torch.from_numpy(a).to(dev)  # noqa: E731
ug = kway.UGraph(t(xadj), t(adj), t(w), t(vw))
for k in (2, 8):
    r = kway.partition_kway(ug, k, tol=0.03, seed=0)
    print(k, r.cut, r.levels)
torch.cuda.synchronize()
