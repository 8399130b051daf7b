"""DOT ingestion on the device (hs_dot_parse, graphio.py:79-199).

* every text of tests/golden/dot_cases.json (outputs of the REFERENCE's own
  parse_dot: its test strings, emitted graphs, hand-written edge cases and
  seeded mutations) gives the reference's graph or exception through the
  drop-in parse_dot;
* seeded mutations generated here agree with the CPU restatement
  (oracle/dot_oracle.py, pinned to the same goldens);
* parse_dot_csr builds the device CSR the object model lowers to, and at
  100k tasks / ~300k edges round-trips emit_dot exactly.
"""
import json
import os
import random

import numpy as np
import pytest
import torch

from oracle import dot_oracle as D

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
with open(os.path.join(HERE, "golden", "dot_cases.json")) as f:
    CASES = json.load(f)["cases"]


def fx(x):
    return "nan" if x != x else float.hex(x)


def result(text):
    from paper_1502_07451_b200.graphio import parse_dot
    try:
        g = parse_dot(text)
    except Exception as exc:  # noqa: BLE001 - compared with the reference's exception
        return {"error": type(exc).__name__, "msg": str(exc)}
    return {"name": g.name, "root": g.root,
            "nodes": [[n.id, n.kind, n.size, fx(n.weight_cpu), fx(n.weight_gpu),
                       [list(p) for p in n.attrs]] for n in g.nodes.values()],
            "edges": [[e.src, e.dst, e.bytes, fx(e.weight_xfer), [list(p) for p in e.attrs]]
                      for e in g.edges.values()]}


@pytest.mark.parametrize("lo", range(0, 900, 150))
def test_parse_dot_matches_reference_goldens(lo):
    for c in CASES[lo:lo + 150]:
        exp = {k: v for k, v in c.items() if k != "text"}
        assert result(c["text"]) == exp, repr(c["text"][:300])


def test_reference_test_module_cases():
    """pkg/tests/test_graphio.py's parse_dot assertions, through the drop-in."""
    from paper_1502_07451_b200.graphio import DotParseError, emit_dot, parse_dot
    g = parse_dot("digraph g { a -> b; }")
    assert g.root == 0 and g.n_kernels() == 2
    g = parse_dot('digraph g { a [weight_cpu=5.0, weight_gpu=1.0]; a -> b; }')
    a = g.nodes[1]
    assert (a.weight_cpu, a.weight_gpu) == (5.0, 1.0)
    with pytest.raises(DotParseError, match="undirected"):
        parse_dot("graph g { a -- b; }")
    with pytest.raises(DotParseError, match="line 3"):
        parse_dot('digraph g {\n a -> b;\n ]]junk!![[;\n}')
    with pytest.raises(DotParseError):
        parse_dot("digraph g { a -> b;")
    g = parse_dot('digraph g { a [shape=box, kind=MA]; a -> b [label="x"]; }')
    assert parse_dot(emit_dot(g)).structurally_equal(g)


ALPHABET = list('ab01n_ .;[]=,"\\-><{}#/\t\r\n') + [" ", "é", "　", " "]


def _mutants(n, seed):
    from paper_1502_07451_b200.gen import generate_random_dag
    from paper_1502_07451_b200.graphio import emit_dot
    rng = random.Random(seed)
    base = [c["text"] for c in CASES if "error" not in c and len(c["text"]) < 4000]
    for s in range(6):
        base.append(emit_dot(generate_random_dag(12 + 5 * s, 20 + 8 * s, "MM", 64, s)))
    out = []
    for _ in range(n):
        t = list(rng.choice(base))
        lo = "".join(t).find("{") + 1
        for _ in range(rng.randint(1, 4)):
            i = rng.randrange(min(lo, len(t)), len(t) + 1)
            r = rng.random()
            if r < 0.45 or not t:
                t.insert(i, rng.choice(ALPHABET))
            elif r < 0.85:
                del t[min(i, len(t) - 1)]
            else:
                t[min(i, len(t) - 1)] = rng.choice(ALPHABET)
        out.append("".join(t))
    return out


def test_mutations_match_oracle():
    for text in _mutants(1500, 11):
        assert result(text) == D.parse(text), repr(text[:300])


def _csr_of_graph(g):
    from paper_1502_07451_b200.csr import HostDag
    h = HostDag.from_taskgraph(g)
    return h


def test_parse_dot_csr_matches_object_model():
    from paper_1502_07451_b200.graphio import parse_dot, parse_dot_csr
    texts = [c["text"] for c in CASES if "error" not in c]
    texts.append("digraph g { n7 -> n3; n3 -> n9; a -> n3; n7 -> n3 [bytes=4]; }")
    from paper_1502_07451_b200._native import NativeError
    for text in texts:
        g = parse_dot(text)
        try:
            h = _csr_of_graph(g)
        except OverflowError:  # bytes beyond int64: a Python int, no CSR form
            with pytest.raises(NativeError, match="int64"):
                parse_dot_csr(text)
            continue
        csr = parse_dot_csr(text)
        assert csr.n == h.n and csr.m == h.m, text[:200]
        assert csr.root == h.root
        assert (csr.ids == h.ids).all()
        assert (csr.out_ptr.cpu().numpy() == h.out_ptr()).all()
        assert (csr.out_dst.cpu().numpy() == h.dst).all()
        for a, b in ((csr.w_cpu, h.w_cpu), (csr.w_gpu, h.w_gpu), (csr.w_xfer, h.w_xfer)):
            assert a.cpu().numpy().tobytes() == np.ascontiguousarray(b).tobytes()
        assert (csr.bytes.cpu().numpy() == h.bytes).all()


def test_parse_dot_csr_large_roundtrip():
    """100k kernels: emit_dot -> parse_dot_csr reproduces the graph's CSR."""
    from paper_1502_07451_b200.costs import SyntheticCostModel
    from paper_1502_07451_b200.gen import generate_random_dag
    from paper_1502_07451_b200.graph import attach_weights
    from paper_1502_07451_b200.graphio import emit_dot, parse_dot_csr
    g = attach_weights(generate_random_dag(100_000, 190_000, "MA", 512, 3), SyntheticCostModel())
    text = emit_dot(g)
    h = _csr_of_graph(g)
    csr = parse_dot_csr(text)
    assert csr.n == h.n and csr.m == h.m and csr.root == h.root
    assert (csr.ids == h.ids).all()
    assert (csr.out_dst.cpu().numpy() == h.dst).all()
    assert csr.w_xfer.cpu().numpy().tobytes() == h.w_xfer.tobytes()
    assert csr.w_gpu.cpu().numpy().tobytes() == h.w_gpu.tobytes()
    # the device CSR runs the hot path: same validate() as the object model
    assert csr.validate() == []


def test_long_literals_exact_on_device():
    """> 19 significant digits whose two Eisel-Lemire bounds differ are decided
    on the device (big-integer midpoint comparison); only int(float()) values
    beyond int64 (Python ints) go to the host."""
    from paper_1502_07451_b200 import _native
    from paper_1502_07451_b200.graphio import parse_dot
    lit = "1.00000000000000011102230246251565404236316680908203125"
    text = f"digraph g {{ a [weight_cpu={lit}]; a -> b [bytes=1e20]; }}"
    info, h = _native.dot_parse(text.encode())
    assert info.status == 0 and info.n_slow == 1  # only the bytes value
    h.close()
    g = parse_dot(text)
    assert g.nodes[1].weight_cpu == float(lit)
    assert g.edges[(1, 2)].bytes == 10 ** 20
