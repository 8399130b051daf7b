"""Phase times of partition_dag on the config-4 DAG under a random numbering
(the band start in longest-path level order), each phase bracketed by CUDA
events after a warm-up call."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1502_07451_b200 import _native, kway

csr = kway.layered_dag(10_000_000, 100_000_000, 0)
rel, _ = kway.relabeled_dag(csr, seed=1)
del csr
torch.cuda.empty_cache()


def phases():
    t = {}
    ev = [torch.cuda.Event(enable_timing=True)]
    ev[0].record()

    def mark(name):
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        ev.append(e)
        t[name] = len(ev) - 1
    ew = kway.integer_weights(rel.w_xfer); nw = kway.integer_weights(rel.w_gpu); mark("integer_weights")
    ug = kway.symmetrize(rel, ew, nw); mark("symmetrize")
    topo = _native.dag_is_topological(rel); mark("is_topological")
    lv, _, _, nl = _native.levels(rel, 0); mark("levels")
    perm, inv = _native.level_permutation(rel, lv, nl); mark("level_permutation")
    pg = kway.permute_ugraph(ug, perm, inv); mark("permute_ugraph")
    r = kway.partition_kway(pg, 8, None, 0.03, 0); mark("partition_kway")
    part = _native.parts_unpermute(perm, r.part, torch.empty_like(r.part)); mark("unpermute")
    torch.cuda.synchronize()
    prev = 0
    out = {}
    for name, i in t.items():
        out[name] = ev[prev].elapsed_time(ev[i])
        prev = i
    out["total"] = ev[0].elapsed_time(ev[-1])
    out["cut"] = r.cut
    return out


phases()
for _ in range(2):
    print({k: (round(v, 3) if isinstance(v, float) else v) for k, v in phases().items()}, flush=True)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(3):
    r = kway.partition_dag(rel, 8, tol=0.03)
b.record()
torch.cuda.synchronize()
print("partition_dag relabelled", a.elapsed_time(b) / 3, "ms cut", r.cut, flush=True)
