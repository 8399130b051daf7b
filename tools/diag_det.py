"""Determinism / weight-scale identity diagnostics for the k-way partitioner."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import torch
from paper_1502_07451_b200 import kway
import _kway_cases as KC

csr = kway.layered_dag(20000, 200000, 4)
ew = torch.full((csr.m,), 37, dtype=torch.int32, device=csr.device)
ug = kway.symmetrize(csr, ew)
os.environ["HS_KWAY_WEIGHTS"] = "1"
ugw = kway.symmetrize(csr, ew)
del os.environ["HS_KWAY_WEIGHTS"]
rs = [kway.partition_kway(ug, 8, tol=0.03, seed=3) for _ in range(3)]
rw = [kway.partition_kway(ugw, 8, tol=0.03, seed=3) for _ in range(3)]
print("unit cuts", [r.cut for r in rs], "levels", [r.levels for r in rs])
print("wgt  cuts", [r.cut for r in rw], "levels", [r.levels for r in rw])
print("unit det", all((r.part == rs[0].part).all().item() for r in rs))
print("wgt det", all((r.part == rw[0].part).all().item() for r in rw))
print("unit==wgt", (rs[0].part == rw[0].part).all().item())
dev = torch.device("cuda")
c = KC.cases()["L500"]()
xadj, adj, w, vw = KC.csr(c)
t = lambda a: torch.from_numpy(a).to(dev)
u5 = kway.UGraph(t(xadj), t(adj), t(w), t(vw))
for rsf in (False, True):
    out = [kway.partition_kway(u5, 2, tol=0.03, seed=0, reference_start=rsf) for _ in range(3)]
    print("L500 k=2 start", rsf, [KC.int_cut(c, r.part.cpu().numpy()) for r in out],
          [r.levels for r in out])
