"""The CPU restatement of parse_dot (oracle/dot_oracle.py) against the
REFERENCE's own outputs (tests/golden/dot_cases.json, made by
tests/golden/make_dot_golden.py from graphio.py:79-199), and the host build of
the device's float() conversion (hs_dot_py_float) against CPython's float()."""
import json
import os
import random
import struct

import pytest

from oracle import dot_oracle as D

HERE = os.path.dirname(os.path.abspath(__file__))
with open(os.path.join(HERE, "golden", "dot_cases.json")) as f:
    CASES = json.load(f)["cases"]


def expected(c):
    return {k: v for k, v in c.items() if k != "text"}


def test_golden_corpus_shape():
    assert len(CASES) > 800
    kinds = {c.get("error", "ok") for c in CASES}
    assert {"ok", "DotParseError", "ValueError", "OverflowError"} <= kinds
    msgs = " ".join(c.get("msg", "") for c in CASES)
    for m in ("expected a digraph header", "undirected", "cannot parse statement",
              "bad attribute syntax", "no digraph found", "missing closing brace"):
        assert m in msgs


@pytest.mark.parametrize("lo", range(0, 900, 100))
def test_oracle_matches_reference(lo):
    for c in CASES[lo:lo + 100]:
        assert D.parse(c["text"]) == expected(c), repr(c["text"][:200])


def _py_float_cases(n, seed):
    rng = random.Random(seed)
    out = ["0", "-0", "1.5", ".5", "5.", "1e5", "1E-5", " 3.25\t", "inf", "-Infinity", "nan",
           "1_000", "1__0", "_1", "1_", "1._5", "1e1_0", "abc", "", ".", "e5", "1e", "+.5e-3",
           "4.9e-324", "2.4703282292062328e-324", "1.7976931348623157e308",
           "1.7976931348623159e308", "9007199254740993", "1e400", "1e-400", " 1 "]
    for _ in range(n):
        k = rng.random()
        if k < 0.4:
            out.append(repr(struct.unpack("<d", struct.pack("<Q", rng.getrandbits(64)))[0]))
        elif k < 0.7:
            out.append("%.*e" % (rng.randint(0, 18), rng.uniform(0, 10) * 10 ** rng.randint(-320, 308)))
        else:
            out.append(f"{rng.randint(0, 10 ** 17)}.{rng.randint(0, 10 ** 8)}e{rng.randint(-340, 320)}")
    return out


def test_device_float_restatement_matches_cpython():
    """hs_dot_py_float is the device's conversion compiled for the host: every
    literal converts bit-exactly or is rejected as float() rejects it."""
    from paper_1502_07451_b200 import _native as N
    for s in _py_float_cases(20000, 7):
        st, v = N.dot_py_float(s.encode())
        try:
            ref = float(s)
        except ValueError:
            assert st == 1, s
            continue
        assert st == 0, s
        assert struct.pack("<d", v) == struct.pack("<d", ref) or (v != v and ref != ref), s


def _halfway_literals(n, seed):
    """Decimal literals at and around the exact midpoint of two adjacent doubles,
    written with 20 to 800 significant digits (the big-integer path)."""
    import math
    from decimal import Decimal, getcontext
    getcontext().prec = 1200
    rng = random.Random(seed)
    out = []
    for _ in range(n):
        k = rng.random()
        if k < 0.1:
            x = struct.unpack("<d", struct.pack("<Q", rng.getrandbits(52)))[0]  # subnormal
        else:
            x = abs(struct.unpack("<d", struct.pack("<Q", rng.getrandbits(63)))[0])
        if not math.isfinite(x):
            continue
        y = math.nextafter(x, math.inf)
        if not math.isfinite(y):
            continue
        mid = (Decimal(x) + Decimal(y)) / 2
        txt = format(mid, "f") if rng.random() < 0.5 else format(mid, "e")
        out.append(txt)
        sig = "".join(c for c in format(mid, "e").split("e")[0] if c.isdigit())
        ex = int(format(mid, "e").split("e")[1])
        for nd in (20, 25, 40, len(sig)):
            if nd <= len(sig):
                t = sig[:nd]
                out.append(f"{t[0]}.{t[1:]}e{ex}")
                out.append(f"{t[0]}.{t[1:]}1e{ex}")  # just above a truncated midpoint
    return out


def test_device_float_long_literals_exact():
    """> 19 significant digits (midpoints of adjacent doubles and their
    neighbours): the big-integer comparison rounds like CPython."""
    from paper_1502_07451_b200 import _native as N
    for s in _halfway_literals(400, 3):
        st, v = N.dot_py_float(s.encode())
        ref = float(s)
        assert st == 0, s
        assert struct.pack("<d", v) == struct.pack("<d", ref), (s[:80], v, ref)
