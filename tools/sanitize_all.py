"""Small invocations of every hot-path kernel family for compute-sanitizer
(memcheck / racecheck / synccheck): k-way (CTA FM levels and Jet levels),
K1/K2/K7 (dataflow and frontier), device topological order, validation,
weights, DES with trace products, batched generator, exact 2-way FM, DOT
ingestion (every golden text plus the device CSR of the emitted graphs)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch
import paper_1502_07451_b200 as H
from paper_1502_07451_b200 import gen, kway, sim
from paper_1502_07451_b200.graph import topological_order, validate
import _kway_cases as KC
from _util import random_weighted_graph

dev = torch.device("cuda")
c = KC.cases()["L200"]()
xadj, adj, w, vw = KC.csr(c)
t = lambda a: torch.from_numpy(a).to(dev)  # noqa: E731
ug = kway.UGraph(t(xadj), t(adj), t(w), t(vw))
for k in (2, 8):
    print("fm", k, kway.partition_kway(ug, k, seed=0).cut)
csr = kway.layered_dag(6000, 40000, seed=1)
print("jet", kway.partition_dag(csr, 8).cut)
rel, _ = kway.relabeled_dag(csr, 1)
print("levels", kway.levels(csr)[2], kway.levels(rel)[2])
parts = torch.randint(0, 4, (1, csr.n), dtype=torch.int32, device=dev)
print("evaluate", kway.evaluate_batch(csr, parts, 4)["cut_edges"][0].item())
g = random_weighted_graph(5, max_kernels=30)
print("topo", topological_order(g)[:5], validate(g))
tr = sim.simulate(g, H.build_policy("dmda", g), sim.MachineModel(3, 1))
print("sim", sim.metrics(tr)["makespan"], len(sim.trace_csv(tr)))
print("heuristic", H.partition_heuristic(g, H.workload_ratio(g)).edge_cut)
b = gen.generate_random_dag_batch(38, 75, "MA", 1024, range(64))
print("rgen", int(b.edge_counts.sum()))
print("compare", sim.compare(["gp"], gen.RandomDagFactory(38, 75), iterations=16)[0].mean_makespan)
import json
from paper_1502_07451_b200.graphio import parse_dot, parse_dot_csr
with open(os.path.join(ROOT, "tests", "golden", "dot_cases.json")) as f:
    cases = json.load(f)["cases"]
ok = 0
for cse in cases:
    try:
        parse_dot(cse["text"])
        if "error" not in cse:
            parse_dot_csr(cse["text"])
        ok += 1
    except Exception:  # noqa: BLE001 - the expected parse errors
        pass
print("dot", ok, len(cases))
torch.cuda.synchronize()
print("done")
