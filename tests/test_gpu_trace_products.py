"""Trace products against the REFERENCE (sim.py:200-331, graphio.py:221-270).

tests/golden/trace_products.json holds, for 21 golden graphs x 3 machines x
3 policies, the reference's metrics(trace) and the sha256 of trace_csv,
annotated_dot and emit_dot (tests/golden/make_trace_golden.py, run on the
unmodified reference). Checked here:

* simulate()'s event order comes from the device sort (hs_trace_sort) and
  reproduces trace_csv byte for byte;
* metrics() reduced on the device (hs_trace_metrics) equals the reference's
  dict exactly, and equals the host loop over the same events;
* annotated_dot / emit_dot text is byte-identical;
* the device order equals the reference's sort key on large traces too
  (ids past 9 digits' string order, many workers: "cpu10" < "cpu2").
"""
import hashlib
import json
import os

import numpy as np
import pytest

from _util import graph_from_spec

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
with open(os.path.join(HERE, "golden", "trace_products.json")) as f:
    GOLD = json.load(f)["cases"]
with open(os.path.join(HERE, "golden", "small_graphs.json")) as f:
    SPECS = {c["name"]: c["spec"] for c in json.load(f)}
with open(os.path.join(HERE, "golden", "medium_graphs.json")) as f:
    SPECS.update({c["name"]: c["spec"] for c in json.load(f)})


def sha(t):
    return hashlib.sha256(t.encode()).hexdigest()


@pytest.mark.parametrize("case", GOLD, ids=[c["name"] for c in GOLD])
def test_trace_products_match_reference(case):
    from paper_1502_07451_b200.graphio import emit_dot
    from paper_1502_07451_b200.policies import build_policy
    from paper_1502_07451_b200 import sim
    g = graph_from_spec(SPECS[case["name"]])
    assert sha(emit_dot(g)) == case["emit_dot_sha256"]
    if "emit_dot" in case:
        assert emit_dot(g) == case["emit_dot"]
    for key, want in case["sims"].items():
        pol, c, w = key.split("_")
        tr = sim.simulate(g, build_policy(pol, g), sim.MachineModel(int(c), int(w)))
        assert sha(sim.trace_csv(tr)) == want["trace_sha256"], key
        m = sim.metrics(tr)
        assert m == want["metrics"], key
        host = sim.metrics(sim.Trace(list(tr.events), tr.makespan, tr.transfer_count,
                                     tr.transfer_bytes, tr.busy_ms, tr.kernels_per_device))
        assert host == m, key
        ad = sim.annotated_dot(g, tr)
        assert sha(ad) == want["annotated_dot_sha256"], key
        if want["annotated_dot"] is not None:
            assert ad == want["annotated_dot"]


def _ref_key_order(raw, ids, names):
    """The reference's sort key (sim.py:200) applied to device records."""
    order = {0: 0, 1: 1, 2: 2, 3: 3}
    keys = []
    for i, r in enumerate(raw):
        a, b, k = int(r["a"]), int(r["b"]), int(r["kind"])
        if k >= 2:
            subj, res = str(int(ids[a])), names[int(r["resource"])]
        else:
            subj = f"d{int(ids[a])}.{int(ids[b])}" if b >= 0 else f"d{int(ids[a])}"
            res = "bus"
        keys.append((float(r["time"]), order[k], subj, res, i))
    return [t[-1] for t in sorted(keys)]


def test_device_sort_matches_reference_key_on_synthetic_events():
    """Random event records with colliding times, ids across digit counts and
    12 CPU workers (string order of names): hs_trace_sort == sorted()."""
    import torch
    from paper_1502_07451_b200 import _native, sim
    rng = np.random.default_rng(3)
    n_nodes, cnt = 500, 20000
    big = np.unique(rng.integers(1000, 10 ** 11, 2 * n_nodes))[:n_nodes - 40]
    ids = np.concatenate([np.sort(rng.choice(np.arange(1, 200), 40, replace=False)),
                          big]).astype(np.int64)
    names = [f"cpu{i}" for i in range(12)] + [f"gpu{i}" for i in range(3)]
    raw = np.zeros(cnt, dtype=_native.EVENT_DTYPE)
    raw["time"] = rng.integers(0, 50, cnt) * 0.25
    raw["kind"] = rng.integers(0, 4, cnt)
    raw["a"] = rng.integers(0, n_nodes, cnt)
    raw["b"] = np.where(rng.random(cnt) < 0.5, rng.integers(0, n_nodes, cnt), -1)
    raw["resource"] = np.where(raw["kind"] >= 2, rng.integers(0, len(names), cnt), -1)
    raw["b"] = np.where(raw["kind"] >= 2, -1, raw["b"])
    dev = torch.device("cuda")
    ev = torch.from_numpy(raw.view(np.uint8).copy()).to(dev)
    perm = _native.trace_sort(ev, cnt, torch.from_numpy(ids).to(dev),
                              torch.tensor(sim._resource_ranks(names), dtype=torch.int32,
                                           device=dev))
    assert perm.cpu().numpy().tolist() == _ref_key_order(raw, ids, names)


def test_large_trace_metrics_match_host_loop():
    """A 3,000-kernel DAG under 12 CPU + 2 GPU workers: device order and
    metrics equal the host sort/loop over the same device records."""
    from paper_1502_07451_b200 import gen, sim
    from paper_1502_07451_b200.costs import SyntheticCostModel
    from paper_1502_07451_b200.graph import attach_weights
    from paper_1502_07451_b200.policies import build_policy
    g = attach_weights(gen.generate_random_dag(3000, 6000, "MA", 512, seed=4), SyntheticCostModel())
    for pol in ("eager", "dmda"):
        tr = sim.simulate(g, build_policy(pol, g), sim.MachineModel(12, 2))
        ev = list(tr.events)
        assert ev == sorted(ev, key=lambda e: (e.time, sim.EVENT_ORDER[e.kind], e.subject,
                                               e.resource))
        host = sim.metrics(sim.Trace(ev, tr.makespan, tr.transfer_count, tr.transfer_bytes,
                                     tr.busy_ms, tr.kernels_per_device))
        assert sim.metrics(tr) == host
        assert host["makespan"] == tr.makespan and host["transfer_count"] == tr.transfer_count
