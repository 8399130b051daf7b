"""Task graphs for the validate / topological_order goldens (test infrastructure).

Plain specs ({"root", "nodes": [[id, kind, size, w_cpu, w_gpu]], "edges":
[[u, v, bytes, w_xfer]]}) so the golden script can build them with the
REFERENCE's classes (tests/golden/make_validate_golden.py) and the tests with
the drop-in's. Crafted invalid graphs (self-loops, cycles, negative weights,
kernels without predecessors, weighted roots, ids not starting at 0, a root
that is not the smallest id) plus seeded random DAGs with arbitrary id
numbering and seeded random graphs closed into cycles.
"""
from __future__ import annotations

import random

SOURCE = "SOURCE"


def _spec(nodes, edges, root=0):
    ns = [[root, SOURCE, 0, 0.0, 0.0]] + [[i, "K", 64, wc, wg] for i, wc, wg in nodes]
    return {"root": root, "nodes": ns, "edges": [list(e) for e in edges]}


CRAFTED = {
    "valid_chain": ([(1, 1.0, 1.0), (2, 1.0, 1.0)], [(0, 1, 0, 0.0), (1, 2, 8, 0.5)]),
    "self_loop": ([(1, 1.0, 1.0), (2, 1.0, 1.0)], [(0, 1, 0, 0.0), (1, 2, 8, 0.5), (2, 2, 8, 0.5)]),
    "cycle": ([(1, 1.0, 1.0), (2, 1.0, 1.0), (3, 1.0, 1.0), (4, 1.0, 1.0)],
              [(0, 1, 0, 0.0), (1, 2, 8, 0.5), (2, 3, 8, 0.5), (3, 2, 8, 0.5), (3, 4, 8, 0.5)]),
    "two_cycles": ([(i, 1.0, 1.0) for i in range(1, 8)],
                   [(0, 1, 0, 0.0), (1, 2, 1, 0.1), (2, 3, 1, 0.1), (3, 2, 1, 0.1),
                    (1, 5, 1, 0.1), (5, 6, 1, 0.1), (6, 7, 1, 0.1), (7, 5, 1, 0.1),
                    (0, 4, 0, 0.0)]),
    "negative": ([(1, -1.0, 1.0), (2, 1.0, -2.0)], [(0, 1, 0, 0.0), (1, 2, -8, -0.5)]),
    "no_root_edge": ([(1, 1.0, 1.0), (2, 1.0, 1.0), (3, 1.0, 1.0)], [(0, 1, 0, 0.0)]),
    "many": ([(1, -1.0, 1.0), (2, 1.0, 1.0), (3, 1.0, 1.0)],
             [(1, 1, 0, -1.0), (1, 2, 8, 0.5), (2, 1, 8, 0.5), (3, 3, -1, 0.1)]),
    "wide_ids": ([(10, 1.0, 1.0), (7, 1.0, 1.0), (42, 1.0, 1.0), (3, 1.0, 1.0)],
                 [(0, 42, 0, 0.0), (42, 7, 4, 0.1), (42, 3, 4, 0.1), (3, 10, 4, 0.1),
                  (7, 10, 4, 0.1)]),
    "diamond_ties": ([(i, 1.0, 1.0) for i in range(1, 7)],
                     [(0, 5, 0, 0.0), (0, 6, 0, 0.0), (5, 2, 1, 0.1), (6, 1, 1, 0.1),
                      (2, 3, 1, 0.1), (1, 3, 1, 0.1), (3, 4, 1, 0.1)]),
}


def _root_weighted():
    s = _spec([(1, 1.0, 1.0)], [(0, 1, 0, 0.0)])
    s["nodes"][0] = [0, SOURCE, 0, 1.0, 0.0]
    return s


def _root_mid():
    # the root is not the smallest id: kernels 1..3 below it, 5..6 above
    s = _spec([(1, 1.0, 1.0), (2, 1.0, 1.0), (3, 1.0, 1.0), (5, 1.0, 1.0), (6, 1.0, 1.0)],
              [(4, 3, 0, 0.0), (4, 6, 0, 0.0), (3, 1, 2, 0.1), (6, 2, 2, 0.1), (1, 5, 2, 0.1),
               (2, 5, 2, 0.1)], root=4)
    return s


def random_dag_spec(seed, n, m, permute=True, cycle=False):
    """A random DAG (edges from lower to higher creation index), node ids a
    random permutation of a sparse id range; cycle=True adds one back edge."""
    rng = random.Random(seed)
    ids = rng.sample(range(1, 4 * n + 1), n) if permute else list(range(1, n + 1))
    edges = set()
    for _ in range(m):
        a, b = sorted(rng.sample(range(n), 2))
        edges.add((a, b))
    has_pred = {b for _, b in edges}
    out = [(0, ids[i], 0, 0.0) for i in range(n) if i not in has_pred]
    out += [(ids[a], ids[b], rng.randrange(1, 64), round(rng.random(), 3)) for a, b in sorted(edges)]
    if cycle and edges:
        a, b = sorted(edges)[rng.randrange(len(edges))]
        out.append((ids[b], ids[a], 1, 0.1))
    nodes = [(ids[i], round(rng.random() * 5, 3), round(rng.random() * 5, 3)) for i in range(n)]
    return _spec(nodes, out)


def cases():
    for name in sorted(CRAFTED):
        yield name, _spec(*CRAFTED[name])
    yield "root_weighted", _root_weighted()
    yield "root_mid", _root_mid()
    for seed in range(12):
        n = 8 + 7 * seed
        yield f"random_{seed}", random_dag_spec(seed, n, 3 * n)
    for seed in range(8):
        n = 10 + 5 * seed
        yield f"random_cycle_{seed}", random_dag_spec(100 + seed, n, 2 * n, cycle=True)
    yield "random_ordered", random_dag_spec(77, 300, 1200, permute=False)
    yield "random_large", random_dag_spec(78, 2000, 8000)
