"""Golden trace products of the REFERENCE: metrics, annotated_dot, emit_dot,
trace_csv (sim.py:207-331, graphio.py:221-270).

Run here (not on the GPU box, where /root/reference does not exist):

    python tests/golden/make_trace_golden.py

Imports the unmodified reference (read-only, bytecode writing disabled) and,
for the first golden graphs of small_graphs.json / medium_graphs.json under
three machines and the three built-in policies, records metrics(trace), the
sha256 of trace_csv(trace), of annotated_dot(graph, trace) and of
emit_dot(graph) (the full text for small ones) into
tests/golden/trace_products.json.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
HERE = os.path.dirname(os.path.abspath(__file__))

from hetsched.graph import DataEdge, KernelNode, TaskGraph  # noqa: E402
from hetsched.graphio import emit_dot  # noqa: E402
from hetsched.policies import build_policy  # noqa: E402
from hetsched.sim import MachineModel, annotated_dot, metrics, simulate, trace_csv  # noqa: E402


def build(spec):
    nodes = [KernelNode(int(i), k, int(s), float(wc), float(wg)) for i, k, s, wc, wg in spec["nodes"]]
    edges = [DataEdge(int(u), int(v), int(b), float(w)) for u, v, b, w in spec["edges"]]
    return TaskGraph(nodes, edges, root=spec["root"])


def sha(text):
    return hashlib.sha256(text.encode()).hexdigest()


def main():
    with open(os.path.join(HERE, "small_graphs.json")) as f:
        small = json.load(f)
    with open(os.path.join(HERE, "medium_graphs.json")) as f:
        medium = json.load(f)
    cases = [c for c in small[:16]] + [c for c in medium]
    out = {"cases": []}
    for c in cases:
        g = build(c["spec"])
        rec = {"name": c["name"], "emit_dot_sha256": sha(emit_dot(g)), "sims": {}}
        if len(g.nodes) <= 12:
            rec["emit_dot"] = emit_dot(g)
        for (cw, gw) in ((3, 1), (1, 1), (2, 2)):
            for pol in ("eager", "dmda", "gp"):
                tr = simulate(g, build_policy(pol, g), MachineModel(cw, gw))
                ad = annotated_dot(g, tr)
                m = metrics(tr)
                rec["sims"][f"{pol}_{cw}_{gw}"] = {
                    "metrics": m, "trace_sha256": sha(trace_csv(tr)),
                    "annotated_dot_sha256": sha(ad),
                    "annotated_dot": ad if len(g.nodes) <= 8 else None}
        out["cases"].append(rec)
    with open(os.path.join(HERE, "trace_products.json"), "w") as f:
        json.dump(out, f, separators=(",", ":"))
    print("wrote", len(out["cases"]), "graphs")


if __name__ == "__main__":
    main()
