"""Generate golden vectors by running the REFERENCE implementation.

Run here (not on the GPU box, where /root/reference does not exist):

    python tests/golden/make_golden.py

It imports the unmodified reference package from /root/reference/pkg/src
(read-only; bytecode writing disabled) and records its outputs for seeded
inputs into tests/golden/*.json. Floats are stored via json (repr), which
round-trips exactly. The fixtures pin both the oracle (CPU tests) and the
device path (GPU tests).
"""
from __future__ import annotations

import hashlib
import json
import os
import random
import sys

sys.dont_write_bytecode = True
REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

from hetsched.costs import (PartitionTargets, SyntheticCostModel,  # noqa: E402
                            load_calibration, workload_ratio)
from hetsched.graph import (DataEdge, InfeasibleGraphError, KernelNode,  # noqa: E402
                            ROOT_ID, SOURCE_KIND, TaskGraph, attach_weights,
                            generate_random_dag, topological_order, total_weights)
from hetsched.partition import (Partition, PartitionConfig,  # noqa: E402
                                brute_force_partition, evaluate, fm_refine,
                                partition_heuristic)
from hetsched.policies import build_policy  # noqa: E402
from hetsched.sim import (MachineModel, compare, compare_csv,  # noqa: E402
                          critical_path_lower_bound, simulate, trace_csv)

OUT = os.path.dirname(os.path.abspath(__file__))


def random_weighted_graph(seed, max_kernels=15, kind="MA", size=256):
    """Same recipe as the reference's tests/conftest.py:30-40."""
    rng = random.Random(seed)
    n = rng.randint(2, max_kernels)
    m = rng.randint(0, 2 * (n - 1))
    while True:
        try:
            g = generate_random_dag(n, m, kind, size, seed=seed)
            break
        except InfeasibleGraphError:
            m -= 1
    return attach_weights(g, SyntheticCostModel())


def spec_of(g):
    return {"root": g.root,
            "nodes": [[n.id, n.kind, n.size, n.weight_cpu, n.weight_gpu]
                      for n in sorted(g.nodes.values(), key=lambda n: n.id)],
            "edges": [[u, v, e.bytes, e.weight_xfer] for (u, v), e in sorted(g.edges.items())]}


def bits(p: Partition, g):
    return "".join("0" if p.assignment[i] == "CPU" else "1" for i in g.kernel_ids())


def part_record(p: Partition, g):
    return {"assign": bits(p, g), "edge_cut": p.edge_cut, "balance_error": p.balance_error,
            "feasible": p.feasible, "side_weights": list(p.side_weights)}


def sim_record(trace):
    csv = trace_csv(trace)
    return {"makespan": trace.makespan, "transfer_count": trace.transfer_count,
            "transfer_bytes": trace.transfer_bytes,
            "busy": [trace.busy_ms["CPU"], trace.busy_ms["GPU"]],
            "kpd": [trace.kernels_per_device["CPU"], trace.kernels_per_device["GPU"]],
            "trace_sha256": hashlib.sha256(csv.encode()).hexdigest(),
            "trace_csv": csv if len(csv) < 6000 else None}


def graph_case(g, name, brute=True, tol_loose=0.25, machines=((3, 1), (1, 1), (2, 2))):
    ids = g.kernel_ids()
    rec = {"name": name, "spec": spec_of(g)}
    rec["topological_order"] = topological_order(g)
    rec["total_weights"] = list(total_weights(g))
    t = workload_ratio(g)
    rec["workload_ratio"] = t.r_cpu
    rec["critical_path"] = critical_path_lower_bound(g)
    half = PartitionTargets(0.5, 0.5)
    rec["heuristic_half"] = part_record(partition_heuristic(g, half), g)
    rec["heuristic_ratio"] = part_record(partition_heuristic(g, t), g)
    rec["heuristic_loose_seed1"] = part_record(
        partition_heuristic(g, PartitionTargets(0.4, 0.6),
                            PartitionConfig(imbalance_tolerance=tol_loose, seed=1)), g)
    rec["heuristic_cpu_source"] = part_record(
        partition_heuristic(g, half, PartitionConfig(node_weight_source="CPU",
                                                     imbalance_tolerance=0.05)), g)
    if brute and len(ids) <= 14:
        rec["brute_half"] = part_record(brute_force_partition(g, half, tol_loose), g)
    cfg = PartitionConfig(imbalance_tolerance=tol_loose)
    alt = {i: ("CPU" if k % 2 else "GPU") for k, i in enumerate(ids)}
    p0 = Partition(dict(alt), 0.0, 0.0, half)
    cut, err, sides = evaluate(g, p0)
    rec["evaluate_alt"] = {"assign": "".join("0" if alt[i] == "CPU" else "1" for i in ids),
                           "edge_cut": cut, "balance_error": err, "side_weights": list(sides)}
    p0.edge_cut, p0.balance_error, p0.side_weights = cut, err, sides
    p0.feasible = err <= tol_loose
    rec["fm_refine_alt"] = part_record(fm_refine(g, p0, half, cfg), g)
    sims = {}
    for (c, gw) in machines:
        for pol in ("eager", "dmda", "gp"):
            trace = simulate(g, build_policy(pol, g), MachineModel(c, gw))
            sims[f"{pol}_{c}_{gw}"] = sim_record(trace)
    rec["simulate"] = sims
    return rec


CHOL_CSV = """kind,size,time_cpu_ms,time_gpu_ms
POTRF,512,6.0,0.9
TRSM,512,11.0,0.45
SYRK,512,11.5,0.42
GEMM,512,22.0,0.6
[transfer]
latency_ms,bandwidth_bytes_per_ms
0.01,12000000.0
"""


def cholesky_graph(tiles):
    """SURVEY App. D construction (mirrors paper_1502_07451_b200.gen.cholesky_dag)."""
    tasks, last, deps = [], {}, set()

    def add(kind, out, inputs):
        tasks.append(kind)
        tid = len(tasks)
        for s in inputs:
            if s:
                deps.add((s, tid))
        last[out] = tid
        return tid

    trsm = {}
    for k in range(tiles):
        p = add("POTRF", (k, k), [last.get((k, k), 0)])
        for i in range(k + 1, tiles):
            trsm[(i, k)] = add("TRSM", (i, k), [p, last.get((i, k), 0)])
        for i in range(k + 1, tiles):
            add("SYRK", (i, i), [trsm[(i, k)], last.get((i, i), 0)])
            for j in range(k + 1, i):
                add("GEMM", (i, j), [trsm[(i, k)], trsm[(j, k)], last.get((i, j), 0)])
    nodes = [KernelNode(ROOT_ID, SOURCE_KIND, 0)]
    nodes += [KernelNode(t + 1, kind, 512) for t, kind in enumerate(tasks)]
    has = {v for (_, v) in deps}
    tile = 512 * 512 * 8
    edges = [DataEdge(u, v, bytes=tile) for (u, v) in sorted(deps)]
    edges += [DataEdge(ROOT_ID, t, bytes=tile) for t in range(1, len(tasks) + 1) if t not in has]
    return attach_weights(TaskGraph(nodes, edges), load_calibration(CHOL_CSV))


def main():
    small = [graph_case(random_weighted_graph(s), f"rwg{s}") for s in range(40)]
    # MM regime and a tighter tolerance family
    small += [graph_case(random_weighted_graph(100 + s, kind="MM", size=1024), f"rwg_mm{s}")
              for s in range(10)]
    with open(os.path.join(OUT, "small_graphs.json"), "w") as f:
        json.dump(small, f)

    medium = []
    for s, (n, m, kind) in enumerate([(38, 75, "MA"), (120, 240, "MA"), (120, 240, "MM"),
                                      (250, 500, "MA")]):
        g = attach_weights(generate_random_dag(n, m, kind, 1024, seed=s), SyntheticCostModel())
        medium.append(graph_case(g, f"gen_{n}_{m}_{kind}", brute=False,
                                 machines=((3, 1), (4, 2))))
    medium.append(graph_case(cholesky_graph(8), "cholesky_T8", brute=False,
                             machines=((3, 1), (8, 1))))
    with open(os.path.join(OUT, "medium_graphs.json"), "w") as f:
        json.dump(medium, f)

    factory = lambda s: attach_weights(  # noqa: E731
        generate_random_dag(38, 75, "MA", 1024, seed=s), SyntheticCostModel())
    rows = compare(["eager", "dmda", "gp"], factory, MachineModel(3, 1), iterations=64, seed=0)
    cmp = {"iterations": 64, "seed": 0,
           "rows": [{k: getattr(r, k) for k in ("policy", "mean_makespan", "sd_makespan",
                                                "mean_transfers", "sd_transfers",
                                                "mean_transfer_bytes")} for r in rows],
           "csv": compare_csv(rows)}
    with open(os.path.join(OUT, "compare_cfg5_64.json"), "w") as f:
        json.dump(cmp, f)
    print("wrote", len(small), "small,", len(medium), "medium cases")


if __name__ == "__main__":
    main()
