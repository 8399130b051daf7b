"""A/B of the k-way partitioner between two builds (argv[1] = package root):
partitions of the quality cases and of the smoke-sized DAG, printed as
(name, k, cut, sha1 of the part array, ms) so two runs can be diffed."""
import hashlib
import os
import sys
import time

sys.path.insert(0, sys.argv[1])
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
import torch  # noqa: E402
from paper_1502_07451_b200 import kway  # noqa: E402
import _kway_cases as KC  # noqa: E402

dev = torch.device("cuda")
names = sys.argv[2].split(",") if len(sys.argv) > 2 else None
ALL = KC.cases()
for name in sorted(ALL):
    if names and name not in names:
        continue
    c = ALL[name]()
    xadj, adj, w, vw = KC.csr(c)
    t = lambda a: torch.from_numpy(a).to(dev)  # noqa: E731
    ug = kway.UGraph(t(xadj), t(adj), t(w), t(vw))
    for k in (2, 4, 8):
        kway.partition_kway(ug, k, tol=0.03, seed=0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = kway.partition_kway(ug, k, tol=0.03, seed=0)
        torch.cuda.synchronize()
        ms = (time.perf_counter() - t0) * 1e3
        h = hashlib.sha1(r.part.cpu().numpy().tobytes()).hexdigest()[:12]
        print(f"{name:16s} k={k} cut {r.cut:10d} {h} {ms:8.2f} ms", flush=True)
for n, m in ((20_000, 200_000), (100_000, 1_000_000)):
    csr = kway.layered_dag(n, m, seed=1)
    ug = kway.symmetrize(csr)
    for k in (8,):
        kway.partition_kway(ug, k, tol=0.03, seed=0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = kway.partition_kway(ug, k, tol=0.03, seed=0)
        torch.cuda.synchronize()
        ms = (time.perf_counter() - t0) * 1e3
        h = hashlib.sha1(r.part.cpu().numpy().tobytes()).hexdigest()[:12]
        print(f"layered{n:<9d} k={k} cut {r.cut:10d} {h} {ms:8.2f} ms", flush=True)
