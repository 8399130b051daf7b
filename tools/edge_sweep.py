"""Edge-case sweep of partition_kway for compute-sanitizer: tiny graphs, k
above n, isolated vertices, zero-weight vertices, k = 1..64."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1502_07451_b200 import kway
dev = torch.device("cuda")


def ug_of(n, edges, vw=None, ew=None):
    rows = [[] for _ in range(n)]
    wr = [[] for _ in range(n)]
    for i, (u, v) in enumerate(edges):
        w = ew[i] if ew else 1
        rows[u].append(v); wr[u].append(w)
        rows[v].append(u); wr[v].append(w)
    xadj = [0]
    for r in rows:
        xadj.append(xadj[-1] + len(r))
    adj = [x for r in rows for x in r]
    w = [x for r in wr for x in r]
    t = lambda a, d: torch.tensor(a, dtype=d, device=dev)  # noqa: E731
    return kway.UGraph(t(xadj, torch.int64), t(adj or [0], torch.int32)[:len(adj)],
                       t(w or [1], torch.int32)[:len(w)],
                       t(vw if vw else [1] * n, torch.int32))


cases = {
    "n1": (1, []), "n2": (2, [(0, 1)]), "n3_iso": (3, [(0, 1)]), "path10": (10, [(i, i + 1) for i in range(9)]),
    "star20": (20, [(0, i) for i in range(1, 20)]), "empty50": (50, []),
}
for name, (n, e) in cases.items():
    for k in (1, 2, 3, 8, 33, 64):
        for vw in (None, [i % 3 for i in range(n)]):
            try:
                r = kway.partition_kway(ug_of(n, e, vw), k, seed=0)
                torch.cuda.synchronize()
                p = r.part.cpu().tolist()
                assert all(0 <= x < k for x in p), (name, k, p)
                print(name, k, "ok", r.cut, r.feasible)
            except Exception as exc:  # noqa: BLE001 — report API errors, crash on device faults
                print(name, k, "error:", type(exc).__name__, str(exc)[:100])
                torch.cuda.synchronize()
print("done")
