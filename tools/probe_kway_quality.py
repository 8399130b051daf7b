"""k-way quality vs the reference heuristic applied recursively (device exact 2-way kernel).

Prints per case and k: baseline cut (recursive.reference_recursive_parts, the
reference's algorithm bit for bit), the partitioner's cut with and without the
baseline as a start, max deviations and times.
"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import torch
from paper_1502_07451_b200 import kway, recursive
import _kway_cases as KC

dev = torch.device("cuda")
only = sys.argv[1:] or None
for name, f in KC.cases().items():
    if only and name not in only:
        continue
    c = f()
    xadj, adj, w, vw = KC.csr(c)
    t = lambda a: torch.from_numpy(a).to(dev)  # noqa: E731
    ug = kway.UGraph(t(xadj), t(adj), t(w), t(vw))
    for k in (2, 4, 8):
        t0 = time.perf_counter()
        base = recursive.reference_recursive_parts(xadj, adj, w, vw, k, [1.0 / k] * k, 0.03)
        tb = time.perf_counter() - t0
        rows = []
        for rs in (False, True):
            kway.partition_kway(ug, k, tol=0.03, seed=0, reference_start=rs)  # warm
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            r = kway.partition_kway(ug, k, tol=0.03, seed=0, reference_start=rs)
            torch.cuda.synchronize()
            ms = (time.perf_counter() - t0) * 1e3
            p = r.part.cpu().numpy()
            rows.append((KC.int_cut(c, p), KC.max_dev(c, p, k), ms, r.levels, r.cut))
        bc = KC.int_cut(c, base)
        print(f"{name:16s} k={k} base {bc:8d} dev {KC.max_dev(c, base, k):.4f} ({tb*1e3:7.1f} ms) | "
              f"native {rows[0][0]:8d} ({rows[0][0]/bc:.4f}) dev {rows[0][1]:.4f} {rows[0][2]:7.1f} ms lv {rows[0][3]} | "
              f"+start {rows[1][0]:8d} ({rows[1][0]/bc:.4f}) dev {rows[1][1]:.4f} {rows[1][2]:7.1f} ms"
              + ("" if rows[1][0] == rows[1][4] else f" CUT MISMATCH {rows[1][4]}"), flush=True)
