"""K7 timing, 2-way evaluate (mode 0) timing, and the band start on relabelled DAGs."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1502_07451_b200 import _native, kway

ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731


def timed(fn, reps=3):
    r = fn()
    torch.cuda.synchronize()
    a, b = ev(), ev()
    a.record()
    for _ in range(reps):
        r = fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps, r


for n, m in ((100_000, 1_000_000), (10_000_000, 100_000_000)):
    csr = kway.layered_dag(n, m, 0)
    ms, (lv, fin, cp, nl) = timed(lambda: kway.levels(csr))
    print(f"n={n}: levels {ms:.3f} ms, {nl} levels, cp {cp!r}", flush=True)
    ms, _ = timed(lambda: kway.level_order(csr))
    print(f"  level_order (incl levels) {ms:.3f} ms", flush=True)
    nk = csr.n - 1
    two = torch.ones((1, nk), dtype=torch.int8, device=csr.device)
    two[0, :nk // 5] = 0
    ms, (c, cw, tot) = timed(lambda: _native.evaluate2(csr, two, 1, 0))
    print(f"  evaluate2 mode0 1 assignment {ms:.3f} ms cut {float(c[0])!r} cpu {float(cw[0])!r}",
          flush=True)
    ms, r0 = timed(lambda: kway.partition_dag(csr, 8, tol=0.03))
    print(f"  partition_dag ordered: {ms:.3f} ms cut {r0.cut} levels {r0.levels}", flush=True)
    ms, rl = timed(lambda: kway.partition_dag(csr, 8, tol=0.03, order="levels"))
    print(f"  partition_dag forced level order: {ms:.3f} ms cut {rl.cut} ({rl.cut / r0.cut:.4f})",
          flush=True)
    rel, pi = kway.relabeled_dag(csr, seed=1)
    ms, rr = timed(lambda: kway.partition_dag(rel, 8, tol=0.03))
    print(f"  relabelled auto: {ms:.3f} ms cut {rr.cut} ({rr.cut / r0.cut:.4f}) feasible {rr.feasible}",
          flush=True)
    ms, ri = timed(lambda: kway.partition_dag(rel, 8, tol=0.03, order="ids"))
    print(f"  relabelled ids: {ms:.3f} ms cut {ri.cut} ({ri.cut / r0.cut:.4f})", flush=True)
    del csr, rel
    torch.cuda.empty_cache()
