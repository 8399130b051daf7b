"""Golden vectors of the METIS wire boundary, made by running the REFERENCE.

    python tests/golden/make_metis_golden.py

Records, for seeded graphs, the reference's emit_metis text (graphio.py:277-304)
and, for crafted partition files, parse_partition_file's result or exception
message (graphio.py:307-330) into tests/golden/metis_io.json. Run here (the
reference does not exist on the GPU box).
"""
from __future__ import annotations

import json
import os
import sys

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

from hetsched.costs import workload_ratio  # noqa: E402
from hetsched.graph import DataEdge, KernelNode, ROOT_ID, SOURCE_KIND, TaskGraph  # noqa: E402
from hetsched.graphio import emit_metis, parse_partition_file  # noqa: E402
from hetsched.partition import PartitionError  # noqa: E402

from make_golden import random_weighted_graph, spec_of  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def main():
    graphs = []
    for seed in range(24):
        g = random_weighted_graph(seed, max_kernels=12 + seed * 3)
        rec = {"spec": spec_of(g)}
        for src in ("GPU", "CPU"):
            rec[f"metis_{src}"] = emit_metis(g, src)
        rec["metis_scale7"] = emit_metis(g, "GPU", scale=7)
        graphs.append(rec)
    # zero weights everywhere: the reference refuses to integerise
    ns = [KernelNode(ROOT_ID, SOURCE_KIND, 0), KernelNode(1, "K", 64), KernelNode(2, "K", 64)]
    zero = TaskGraph(ns, [DataEdge(0, 1), DataEdge(1, 2, bytes=0, weight_xfer=0.0)])
    try:
        emit_metis(zero)
        zero_err = None
    except PartitionError as exc:
        zero_err = str(exc)

    files = []
    g = random_weighted_graph(3, max_kernels=10)
    n = len(g.kernel_ids())
    texts = {
        "plain": "".join(f"{i % 2}\n" for i in range(n)),
        "spaces_blank_lines": "\n".join([" 1 ", "", "0\t"] + [str(i & 1) for i in range(n - 2)]
                                        + ["", "  "]),
        "crlf_no_final_newline": "\r\n".join(str((i // 2) % 2) for i in range(n)),
        "plus_sign_and_leading_zeros": "\n".join(["+1", "00", "-0"] + ["1"] * (n - 3)) + "\n",
        "bad_value": "\n".join(["0", "1", "2"] + ["0"] * (n - 3)) + "\n",
        "negative_value": "\n".join(["0", "-1"] + ["0"] * (n - 2)) + "\n",
        "not_an_integer": "\n".join(["0", "x1"] + ["0"] * (n - 2)) + "\n",
        "float_line": "\n".join(["0", "1.0"] + ["0"] * (n - 2)) + "\n",
        "too_few": "0\n" * (n - 1),
        "too_many": "1\n" * (n + 1),
        "underscore_int": "\n".join(["1_0"] + ["0"] * (n - 1)) + "\n",
        "vertical_tab_and_formfeed": "\x0b".join(["0"] * 2) + "\x0c" + "\n".join(["1"] * (n - 2)),
        "unicode_space_and_separator": " 1 " + "\n".join(["0"] * (n - 1)),
    }
    targets = workload_ratio(g)
    for name, text in texts.items():
        rec = {"name": name, "text": text}
        try:
            p = parse_partition_file(text, g, targets)
            rec["assignment"] = [p.assignment[k] for k in g.kernel_ids()]
            rec["edge_cut"] = p.edge_cut
            rec["balance_error"] = p.balance_error
        except PartitionError as exc:
            rec["error"] = str(exc)
        files.append(rec)
    with open(os.path.join(OUT, "metis_io.json"), "w") as f:
        json.dump({"graphs": graphs, "zero_weights_error": zero_err,
                   "partition_graph": spec_of(g), "partition_files": files}, f)
    print("wrote", len(graphs), "graphs,", len(files), "partition files")


if __name__ == "__main__":
    main()
