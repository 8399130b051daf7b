"""Golden k-way baselines from the REFERENCE partitioner (run here, not on the GPU box).

    python tests/golden/make_kway_golden.py          # writes tests/golden/kway_baselines.json

For every case of tests/_kway_cases.py (integer weights, the graph
``kway.symmetrize`` builds) it runs the unmodified reference
(/root/reference/pkg/src, read-only, bytecode writing disabled):

* k = 2: ``partition_heuristic`` with r_cpu = 1/2, tolerance 0.03, default
  restarts/seed (partition.py:258-295);
* k = 4, 8: the same heuristic applied recursively (split [p0, p1) at the
  middle, CPU side = lower half, r_cpu = 1/2) — the k-way baseline of
  SURVEY.md §8(c).

It records the integer cut, the max |w_p/W - 1/k| and the part of every
vertex, plus the sha256 of the case arrays. Cases run in parallel processes.
"""
from __future__ import annotations

import json
import os
import sys
import time
from concurrent.futures import ProcessPoolExecutor

sys.dont_write_bytecode = True
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

import _kway_cases as KC  # noqa: E402
from hetsched.costs import PartitionTargets  # noqa: E402
from hetsched.graph import DataEdge, KernelNode, ROOT_ID, SOURCE_KIND, TaskGraph  # noqa: E402
from hetsched.partition import CPU, PartitionConfig, partition_heuristic  # noqa: E402

TOL = 0.03
KS = (2, 4, 8)


def task_graph(case, members):
    """Reference TaskGraph of the induced subgraph: kernel id = position + 1."""
    n, eu, ev, ew, vw = case
    mem = set(int(x) for x in members)
    nodes = [KernelNode(ROOT_ID, SOURCE_KIND, 0)]
    nodes += [KernelNode(int(i) + 1, "K", 0, weight_cpu=float(vw[i]), weight_gpu=float(vw[i]))
              for i in sorted(mem)]
    edges = [DataEdge(int(a) + 1, int(b) + 1, bytes=0, weight_xfer=float(w))
             for a, b, w in zip(eu, ev, ew) if int(a) in mem and int(b) in mem]
    has = {e.dst for e in edges}
    edges += [DataEdge(ROOT_ID, int(i) + 1) for i in sorted(mem) if int(i) + 1 not in has]
    return TaskGraph(nodes, edges)


def recursive(case, members, p0, p1, part):
    if p1 - p0 < 2 or len(members) == 0:
        part[members] = p0
        return
    pm = p0 + (p1 - p0) // 2
    r = (pm - p0) / (p1 - p0)
    g = task_graph(case, members)
    p = partition_heuristic(g, PartitionTargets(r, 1.0 - r), PartitionConfig(imbalance_tolerance=TOL))
    left = np.array([i for i in members if p.assignment[int(i) + 1] == CPU], dtype=np.int64)
    right = np.array([i for i in members if p.assignment[int(i) + 1] != CPU], dtype=np.int64)
    recursive(case, left, p0, pm, part)
    recursive(case, right, pm, p1, part)


def run(name):
    """k = 8 recursion; its depth-1 and depth-2 prefixes are the k = 2 and k = 4
    results (every split is r_cpu = 1/2 of a power-of-two range)."""
    case = KC.cases()[name]()
    n = case[0]
    out = {"name": name, "digest": KC.digest(case), "n": n, "results": {}}
    t = time.perf_counter()
    part8 = np.zeros(n, dtype=np.int64)
    recursive(case, np.arange(n, dtype=np.int64), 0, 8, part8)
    secs = time.perf_counter() - t
    for k in KS:
        part = part8 // (8 // k)
        out["results"][str(k)] = {"cut": KC.int_cut(case, part),
                                  "max_dev": KC.max_dev(case, part, k), "part": part.tolist()}
    out["seconds_k8"] = secs
    print(name, {k: (v["cut"], round(v["max_dev"], 4)) for k, v in out["results"].items()},
          round(secs, 1), flush=True)
    return out


def main():
    names = list(KC.cases())
    with ProcessPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        res = list(ex.map(run, sorted(names, key=lambda s: -KC.cases()[s]()[0])))
    res.sort(key=lambda r: names.index(r["name"]))
    with open(os.path.join(HERE, "kway_baselines.json"), "w") as f:
        json.dump({"tol": TOL, "ks": list(KS), "cases": res}, f)


if __name__ == "__main__":
    main()
