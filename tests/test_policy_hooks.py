"""The policy plugin protocol (policies.py:3-5): on_ready / next_for_worker
of the built-in policies driven by hand, as a caller of the reference would,
and the native simulator's rejection of policies that override a hook.
Known answers follow the reference's semantics (policies.py:19-99); no GPU."""
import pytest

from paper_1502_07451_b200.graph import CPU, GPU
from paper_1502_07451_b200.policies import DmdaPolicy, EagerPolicy, GraphPartitionPolicy
from paper_1502_07451_b200.sim import SimulationError, Worker, _policy_id

from _util import make_graph


class _Sim:
    """The attributes a hook may read (sim.py:95-108)."""

    def __init__(self, graph, workers, resident=()):
        self.graph, self.workers, self.bus_free = graph, workers, 0.0
        self._res = set(resident)

    def item_key(self, e):
        return f"d{e.src}.{e.dst}" if e.src == self.graph.root else f"d{e.src}"

    def resident(self, item, node, t):
        return (item, node) in self._res


def _workers(c=3, g=1):
    ws = [Worker(i, CPU, f"cpu{i}") for i in range(c)]
    return ws + [Worker(c + i, GPU, f"gpu{i}") for i in range(g)]


def test_worker_fields():
    w = _workers()
    assert [x.id for x in w] == [0, 1, 2, 3]
    assert [x.mem_node for x in w] == ["host"] * 3 + ["device"]
    assert w[3].free_time == 0.0 and not w[3].busy


def test_eager_fifo():
    p, sim = EagerPolicy(), None
    for k in (3, 1, 2):
        p.on_ready(k, 0.0, sim)
    w = _workers()
    assert [p.next_for_worker(w[3], 0.0, sim), p.next_for_worker(w[0], 0.0, sim)] == [3, 1]
    assert p.next_for_worker(w[1], 0.0, sim) == 2
    assert p.next_for_worker(w[1], 0.0, sim) is None


def test_dmda_min_estimate_and_queues():
    # kernel 1 is 4x faster on the GPU; its input from the root is not resident
    g = make_graph({1: (4.0, 1.0), 2: (1.0, 1.0)}, [(1, 2, 0.5)])
    w = _workers()
    sim = _Sim(g, w, resident={("d0.1", "host"), ("d0.1", "device")})
    p = DmdaPolicy()
    p.on_ready(1, 0.0, sim)
    assert p.est_free == {3: 1.0} and p.est_bus == 0.0
    # kernel 2: input d1 lives nowhere yet -> every worker pays 0.5 on the bus;
    # est = max(free, avail) + dur: cpu0 = 0.5 + 1 = 1.5, gpu = max(1.0, 0.5) + 1 = 2.0
    p.on_ready(2, 0.0, sim)
    assert p.est_free[0] == 1.5 and p.est_bus == 0.5
    assert p.next_for_worker(w[3], 0.0, sim) == 1
    assert p.next_for_worker(w[0], 0.0, sim) == 2
    assert p.next_for_worker(w[1], 0.0, sim) is None


def test_dmda_tie_goes_to_first_worker():
    g = make_graph({1: (1.0, 1.0)}, [])
    w = _workers(2, 1)
    p = DmdaPolicy()
    p.on_ready(1, 0.0, _Sim(g, w, resident={("d0.1", "host"), ("d0.1", "device")}))
    assert list(p.queues) == [0]


def test_gp_pins_and_missing_kernel():
    p = GraphPartitionPolicy({1: GPU, 2: CPU})
    p.on_ready(1, 0.0, None)
    p.on_ready(2, 0.0, None)
    w = _workers()
    assert p.next_for_worker(w[0], 0.0, None) == 2
    assert p.next_for_worker(w[3], 0.0, None) == 1
    with pytest.raises(KeyError):
        p.on_ready(7, 0.0, None)


def test_native_simulator_accepts_builtins_rejects_overrides():
    assert _policy_id(EagerPolicy()) == 0
    assert _policy_id(DmdaPolicy()) == 1
    assert _policy_id(GraphPartitionPolicy({})) == 2

    class Lifo(EagerPolicy):
        def next_for_worker(self, worker, t, sim):
            return self.queue.pop() if self.queue else None

    class Custom:
        def on_ready(self, kid, t, sim):
            pass

    for pol in (Lifo(), Custom()):
        with pytest.raises(SimulationError, match="not supported by native backend"):
            _policy_id(pol)
