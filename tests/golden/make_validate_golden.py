"""Golden messages of the REFERENCE's validate / topological_order (graph.py:113-172).

Run here (not on the GPU box, where /root/reference does not exist):

    python tests/golden/make_validate_golden.py

Imports the unmodified reference package (read-only, bytecode writing
disabled), builds every case of tests/_validate_cases.py with the reference's
own KernelNode/DataEdge/TaskGraph, and records `validate(graph)` and either
`topological_order(graph)` or the CycleError member into
tests/golden/validate.json. The fixture pins the host restatement (CPU tests)
and the device checks hs_validate_dag / hs_topological_order (GPU tests).
"""
from __future__ import annotations

import json
import os
import sys

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

from hetsched.graph import (CycleError, DataEdge, KernelNode, TaskGraph,  # noqa: E402
                            topological_order, validate)

import _validate_cases as VC  # noqa: E402


def build(spec):
    nodes = [KernelNode(int(i), k, int(s), float(wc), float(wg)) for i, k, s, wc, wg in spec["nodes"]]
    edges = [DataEdge(int(u), int(v), int(b), float(w)) for u, v, b, w in spec["edges"]]
    return TaskGraph(nodes, edges, root=spec["root"])


def main():
    out = {"cases": []}
    for name, spec in VC.cases():
        g = build(spec)
        rec = {"name": name, "spec": spec, "validate": validate(g)}
        try:
            rec["topological_order"] = topological_order(g)
        except CycleError as exc:
            rec["cycle_member"] = exc.member
        out["cases"].append(rec)
    with open(os.path.join(HERE, "validate.json"), "w") as f:
        json.dump(out, f, separators=(",", ":"))
    print("wrote", len(out["cases"]), "cases")


if __name__ == "__main__":
    main()
