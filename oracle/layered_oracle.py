"""CPU restatement of the device layered-DAG generator — TEST INFRASTRUCTURE ONLY.

Restates csrc/gen.cu (the config-2/4 family) in numpy-free pure Python for
small n, so tests can check the device generator bit for bit. Same layout as
the reference generator's layers (graph.py:175-177, 222-223).
"""
from __future__ import annotations

MASK = (1 << 64) - 1


def splitmix64(x: int) -> int:
    x = (x + 0x9E3779B97F4A7C15) & MASK
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & MASK
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & MASK
    return x ^ (x >> 31)


def layout(n: int):
    s = 0
    while s * s < n:
        s += 1
    L = min(max(s, 1), n)
    q, r = divmod(n, L)
    first = [1 + l * q + min(l, r) for l in range(L + 1)]
    return L, first


def generate(n: int, m: int, seed: int):
    """Returns (in_lists, edges): in_lists[v] = sorted preds of node v (root 0)."""
    L, first = layout(n)
    size0 = first[1] - 1
    K = n - size0
    base, rem = divmod(m, K)
    preds = {0: []}
    layer = {}
    for l in range(L):
        for v in range(first[l], first[l + 1]):
            layer[v] = l
    key0 = (seed * 0x2545F4914F6CDD1D) & MASK
    for v in range(1, n + 1):
        l = layer[v]
        if l == 0:
            preds[v] = [0]
            continue
        f = base + (1 if v - 1 - size0 < rem else 0)
        avail = first[l] - 1
        f = min(f, avail)
        key = key0 ^ ((v * 0x9E3779B97F4A7C15) & MASK)
        got = []
        a = 0
        while len(got) < f:
            u = 1 + splitmix64((key + a) & MASK) % avail
            if u not in got:
                got.append(u)
            a += 1
        preds[v] = sorted(got)
    edges = sorted((u, v) for v, ps in preds.items() for u in ps)
    return preds, edges, layer
