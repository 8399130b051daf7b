"""Boundary proof: the reference's own test suite against this package.

The unmodified reference tests (tests/reference_suite/, see its README) run in
a scratch directory laid out like the reference repo — a `tests` package with
the vendored files and a `hetsched` package whose submodules ARE this
package's modules — in a child pytest process on the GPU. Every call the
tests make therefore goes through the drop-in API and the CUDA kernels.

All eight vendored modules run, test_graphio.py (DOT parsing on the device,
METIS export, partition files) included; tests/golden/reference_suite_expected.json
lists the expected failures (none) and the minimum pass count.
"""
import hashlib
import json
import os
import re
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SUITE = os.path.join(HERE, "reference_suite")

SHIM = '''"""`hetsched` -> paper_1502_07451_b200, module for module (test infrastructure)."""
import sys

import paper_1502_07451_b200 as _p
from paper_1502_07451_b200 import costs, graph, graphio, partition, policies, sim
from paper_1502_07451_b200 import *  # noqa: F401,F403


for _m in ("costs", "graph", "graphio", "partition", "policies", "sim"):
    sys.modules["hetsched." + _m] = getattr(_p, _m)
__version__ = _p.__version__
'''


def _sha_list():
    text = open(os.path.join(SUITE, "README.md")).read()
    return dict((name, digest) for digest, name in re.findall(r"([0-9a-f]{64})\s+(\S+\.py)", text))


def test_reference_suite(tmp_path):
    shas = _sha_list()
    assert len(shas) == 8
    work = tmp_path / "ref"
    (work / "tests").mkdir(parents=True)
    (work / "hetsched").mkdir()
    for name, digest in shas.items():
        src = os.path.join(SUITE, name)
        assert hashlib.sha256(open(src, "rb").read()).hexdigest() == digest, f"{name} modified"
        shutil.copy(src, work / "tests" / name)
    (work / "tests" / "__init__.py").write_text("")
    (work / "hetsched" / "__init__.py").write_text(SHIM)
    report = tmp_path / "report.txt"
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([str(work), ROOT]),
               PYTHONDONTWRITEBYTECODE="1")
    proc = subprocess.run([sys.executable, "-m", "pytest", "-q", "-rfE", "-p", "no:cacheprovider",
                           "--rootdir", str(work), str(work / "tests")],
                          cwd=str(work), env=env, capture_output=True, text=True, timeout=3000)
    report.write_text(proc.stdout + proc.stderr)
    out = proc.stdout
    failed = sorted(set(re.findall(r"^(?:FAILED|ERROR) (\S+?)(?: - .*)?$", out, re.M)))
    summary = [ln for ln in out.splitlines() if re.search(r"\d+ (passed|failed)", ln)]
    with open(os.path.join(HERE, "golden", "reference_suite_expected.json")) as f:
        expected = json.load(f)
    exp_fail = sorted(expected["expected_failures"])
    record = os.path.join(ROOT, "gpurun_out")
    if os.path.isdir(record):
        with open(os.path.join(record, "reference_suite_report.txt"), "w") as f:
            f.write(out[-20000:])
    assert summary, out[-4000:]
    assert failed == exp_fail, f"unexpected results: {failed}\n{summary[-1]}"
    m = re.search(r"(\d+) passed", summary[-1])
    assert m and int(m.group(1)) >= expected["min_passed"], summary[-1]
