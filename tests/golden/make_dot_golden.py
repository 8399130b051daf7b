"""Golden outputs of the REFERENCE's parse_dot (graphio.py:79-199).

Run here (not on the GPU box, where /root/reference does not exist):

    python tests/golden/make_dot_golden.py

Imports the unmodified reference package (read-only, bytecode writing
disabled) and records, for every text of the corpus below, either the parsed
graph (name, root, nodes and edges in the TaskGraph's insertion order, floats
as float.hex) or the exception (type and message). The corpus: the DOT
strings of the reference's own test_graphio.py, emit_dot / emit_partitioned_dot
/ annotated_dot of seeded random graphs, hand-written edge cases (quoting and
escapes, comments, every str.splitlines terminator, Unicode whitespace,
several statements per line, closing-brace forms, numbered-name clashes,
default-attribute statements, float() literal forms) and seeded byte-level
mutations of valid texts (which reach the error paths). Written to
tests/golden/dot_cases.json; tests/test_dot_oracle.py pins the CPU
restatement (oracle/dot_oracle.py) to it and tests/test_gpu_dot.py the device
parser (hs_dot_parse).
"""
from __future__ import annotations

import json
import os
import random
import sys

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
HERE = os.path.dirname(os.path.abspath(__file__))

from hetsched.costs import SyntheticCostModel  # noqa: E402
from hetsched.graph import attach_weights, generate_random_dag  # noqa: E402
from hetsched.graphio import emit_dot, emit_partitioned_dot, parse_dot  # noqa: E402
from hetsched.partition import partition_heuristic  # noqa: E402
from hetsched.costs import workload_ratio  # noqa: E402
from hetsched.policies import build_policy  # noqa: E402
from hetsched.sim import annotated_dot, simulate  # noqa: E402


def fx(x: float) -> str:
    return "nan" if x != x else float.hex(x)


def result(text: str) -> dict:
    try:
        g = parse_dot(text)
    except Exception as exc:  # noqa: BLE001 - the exception is the expected output
        return {"error": type(exc).__name__, "msg": str(exc)}
    return {"name": g.name, "root": g.root,
            "nodes": [[n.id, n.kind, n.size, fx(n.weight_cpu), fx(n.weight_gpu),
                       [list(p) for p in n.attrs]] for n in g.nodes.values()],
            "edges": [[e.src, e.dst, e.bytes, fx(e.weight_xfer), [list(p) for p in e.attrs]]
                      for e in g.edges.values()]}


REFERENCE_TEST_TEXTS = [  # pkg/tests/test_graphio.py
    "digraph g { a -> b; }",
    'digraph g { a [weight_cpu=5.0, weight_gpu=1.0]; a -> b; }',
    "graph g { a -- b; }",
    'digraph g {\n a -> b;\n ]]junk!![[;\n}',
    "digraph g { a -> b;",
    'digraph g {\n// a comment\n# another\n"my node" -> b;\n}',
    'digraph g { a [shape=box, kind=MA]; a -> b [label="x"]; }',
    "digraph g {\r\n a -> b;\r\n}\r\n",
]

HAND = [
    "", "\n\n", "// only a comment\n", "# hash\n", "digraph", "digraph g", "digraph g {",
    "digraph g {}", "digraph {}", "digraph g {\n}", "strict digraph g {\n a -> b;\n}",
    "strictdigraph g { }", "digraph g { } trailing garbage", "digraph g {\n a -> b;\n}\n junk !!",
    "digraph \"quoted name\" { a; }", "digraph g_1 {\na\n}", "digraph \"g\" {}",
    "digraph g x { }", "digraph g\n{\na -> b\n}", "digraph g {\n  a -> b -> c;\n}",
    "digraph g { a; b; c; a -> c; b -> c }", "digraph g { a -> b; b -> a; }",
    "digraph g { n5; 5; n05; 05 -> n5; x -> 7; }", "digraph g { n0 -> n1; }",
    "digraph g { 0 -> 1; a; }", "digraph g { n3 -> n1; n1 -> n2; q -> n3; }",
    "digraph g { node [shape=box]; edge [color=red]; graph [rankdir=LR]; a -> b; }",
    'digraph g { "node" [x=1]; node -> edge; }',
    'digraph g { "a\\"b" -> "c d"; "a\\"b" [kind=MM]; }',
    'digraph g { "a;b" -> c; d [label="x;y"]; e [label="[;]"]; }',
    'digraph g { a [label="x", kind=GEMM, size=512, weight_cpu=1.5e2, weight_gpu=.25]; }',
    "digraph g { a [size=1e3]; b [size=-2.7]; c [size=+3]; }",
    "digraph g { a [size=inf]; }", "digraph g { a [size=nan]; }",
    "digraph g { a [weight_cpu=inf, weight_gpu=-Infinity]; }",
    "digraph g { a [weight_cpu=NaN]; }", "digraph g { a [weight_cpu=1_000.5]; }",
    "digraph g { a [weight_cpu=1__0]; }", "digraph g { a [weight_cpu=abc]; }",
    'digraph g { a [weight_cpu=" 2.5 "]; }', 'digraph g { a [weight_cpu=" 2.5 "]; }',
    "digraph g { a -> b [bytes=1e20]; }", "digraph g { a -> b [bytes=12.9, weight_xfer=0.1]; }",
    "digraph g { a -> b [bytes=x]; }", "digraph g { a -> b [weight_xfer=1e400]; }",
    "digraph g { a [size=9223372036854775807]; }",
    "digraph g { a [weight_cpu=0.1000000000000000055511151231257827021181583404541015625]; }",
    "digraph g { a [weight_cpu=2.4703282292062327208828439643411068618252990130716238221279284125033775363510437593264991818081799618989828234772285886546332835517796989819938739800539093906315035659515570226392290858392449105184435931802849936536152500319370457678249219365623669863658480757001585769269903706311928279558551332927834338409351978015531246597263579574622766465272827220056374006485499977096599470454020828166226237857393450736339007967761930577506740176324673600968951340535537458516661134223766678604162159680461914467291840300530057530849048765391711386591646239524912623653881879636239373280423891018672348497668235089863388587925628302755995657524455507255189313690836254779186948667994968324049705821028513185451396213837722826145437693412532098591327667236328125e-324]; }",
    "digraph g { a [weight_cpu=1.00000000000000011102230246251565404236316680908203125]; }",
    "digraph g { a [weight_cpu=1.000000000000000111022302462515654042363166809082031251]; }",
    "digraph g { a [kind=SOURCE]; a -> b; }", "digraph g { b -> a; a [kind=SOURCE]; }",
    "digraph g { a [kind=\"SOURCE\"]; b [kind=SOURCE]; a -> c; }",
    "digraph g { a [kind=SOURCE, kind=K]; a -> b; }",
    "digraph g { a [kind=MA]; a [kind=MM, size=3]; a [size=4]; }",
    "digraph g { a [x=1, y=\"2\", x=3, part=CPU, color=red]; a -> b [z=1, kind=q, bytes=2]; }",
    "digraph g { a [=1]; }", "digraph g { a [x]; }", "digraph g { a [x=]; }",
    "digraph g { a [x=1 y=2]; }", "digraph g { a [x=1,, y=2]; }", "digraph g { a [ x = 1 , ]; }",
    "digraph g { a [x=\"unterminated]; }", "digraph g { a [x=\"a\"b]; }",
    "digraph g { a [x=\"a\" b]; }", "digraph g { a [1x=2]; }",
    "digraph g { a [x=1]] ; }", "digraph g { a [x=1] [y=2]; }", "digraph g { a ]; }",
    "digraph g { a -> ; }", "digraph g { -> b; }", "digraph g { a -> b c; }",
    "digraph g { a b; }", "digraph g { a.b -> c.d; 1.5 -> x; }", "digraph g { a-b; }",
    "digraph g { a;; b; ; }", "digraph g {\n a -> b; // trailing comment\n}",
    "digraph g {\n a -> b; # not a comment here\n}", "digraph g {\n  # a comment line\n a;\n}",
    "digraph g { a [url=\"http://x\"]; }", "digraph g {\n a [l=\"x}\"];\n}",
    "digraph g {\n a;\n \"}\"\n}", "digraph g {\n a; }\n b; }\n", "digraph g {\n a }",
    "digraph g {\n a -> b;\n}", "digraph g {\x0b a -> b;\x0c}", "digraph g {\x1c a;\x1d b;\x1e}",
    "digraph g {\r a -> b;\r}", "digraph g { a; }", "digraph g {\x1f a -> b;\x1f}",
    "digraph g {\n　a -> b ;\n}", " digraph g { a;}",
    "digraph g { café -> b; }", "digraph g { \"café\" -> \"ü\"; }",
    "digraph g { a [label=\"éè\"]; a [x=\"€\"]; }",
    "digraph g { a [x=\"é]; }", "digraph g { a [weight_cpu=\"1.5é]; }",
    "digraph g { \"a\\\\\" -> b; }", "digraph g { \"a\\\" -> b; }",
    "digraph g { a [x=\"q\\\"r\", y=\"\\\\\"]; }",
    "digraph g { n99999999999 -> n1; }", "digraph g { n1 -> n3; b; c; n2; }",
    "digraph g {\n  n0 [kind=SOURCE, size=0, weight_cpu=0.0, weight_gpu=0.0];\n  n0 -> n1;\n}",
    "digraph g { a -> b; a -> b [bytes=5]; }",
    "digraph g { a -> a; }",
    "di graph g {}", "DIGRAPH g {}", "digraph{a->b}", "digraph g {a->b}",
    "digraph g { a [x=1]b; }", "digraph g { [x=1]; }", "digraph g { \"\" -> b; }",
]


def emitted(rng: random.Random):
    model = SyntheticCostModel()
    out = []
    for seed in range(24):
        n = rng.randint(1, 30)
        try:
            g = generate_random_dag(n, rng.randint(0, 2 * n), rng.choice(["MM", "MA"]),
                                    rng.choice([16, 64, 512]), seed)
        except Exception:  # noqa: BLE001 - infeasible edge count: draw again
            continue
        g = attach_weights(g, model)
        out.append(emit_dot(g))
        if seed % 3 == 0 and g.n_kernels() > 0:
            try:
                p = partition_heuristic(g, workload_ratio(g))
                out.append(emit_partitioned_dot(g, p))
            except Exception:  # noqa: BLE001
                pass
        if seed % 4 == 1 and g.n_kernels() > 0:
            try:
                tr = simulate(g, build_policy("dmda", g))
                out.append(annotated_dot(g, tr))
            except Exception:  # noqa: BLE001
                pass
    return out


ALPHABET = list('ab01n_ .;[]=,"\\-><{}#/\t\r\n') + [" ", "é", " "]


def mutate(text: str, rng: random.Random) -> str:
    s = list(text)
    lo = text.find("{") + 1 if rng.random() < 0.8 else 0  # mostly inside the body
    for _ in range(rng.randint(1, 3)):
        op = rng.random()
        i = rng.randrange(min(lo, len(s)), len(s) + 1)
        if op < 0.4 or not s:
            s.insert(i, rng.choice(ALPHABET))
        elif op < 0.8:
            del s[min(i, len(s) - 1)]
        else:
            s[min(i, len(s) - 1)] = rng.choice(ALPHABET)
    return "".join(s)


def corpus():
    rng = random.Random(20260417)
    texts = list(REFERENCE_TEST_TEXTS) + list(HAND)
    em = emitted(rng)
    texts += em
    small = [t for t in texts if 0 < len(t) < 3000]
    for _ in range(700):
        texts.append(mutate(rng.choice(small), rng))
    return texts


def main():
    cases = [{"text": t, **result(t)} for t in corpus()]
    path = os.path.join(HERE, "dot_cases.json")
    with open(path, "w") as f:
        json.dump({"cases": cases}, f, ensure_ascii=True, separators=(",", ":"))
    n_err = sum("error" in c for c in cases)
    print(path, len(cases), "cases", n_err, "errors", os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
