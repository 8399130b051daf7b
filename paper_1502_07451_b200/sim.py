"""Deterministic CPU+GPU machine simulation (drop-in mirror of ``hetsched.sim``).

``simulate`` and ``compare`` run the event loop on the device (K8,
csrc/des.cu): one thread per simulation, bit-exact with the reference because
the loop only adds and maxes fp64 times in the reference's order.
``compare`` packs every iteration's graph into one batch and launches one
kernel per policy instead of looping simulations in Python. The trace
formatting helpers (``trace_csv``, ``compare_csv``, ``metrics``) stay on the
host: they format a finished event list.

Reference: /root/reference/pkg/src/hetsched/sim.py (cited per symbol).
"""
from __future__ import annotations

import io
import statistics
from dataclasses import dataclass
from typing import Callable, Dict, List, Optional, Sequence, Tuple

import numpy as np
import torch

from . import _native
from .csr import DagBatch
from .graph import CPU, GPU, TaskGraph, topological_order, validate, CycleError

HOST = "host"
DEVICE = "device"
EVENT_ORDER = {"xfer_start": 0, "xfer_end": 1, "kernel_start": 2, "kernel_end": 3}
_KIND_NAMES = ("xfer_start", "xfer_end", "kernel_start", "kernel_end")


class SimulationError(Exception):
    """sim.py:23"""


@dataclass(frozen=True)
class MachineModel:
    """C CPU workers (ids 0..C-1) then G GPU workers (sim.py:27-36)."""
    cpu_workers: int = 3
    gpu_workers: int = 1

    def __post_init__(self):
        if self.cpu_workers < 0 or self.gpu_workers < 0:
            raise SimulationError("worker counts must be nonnegative")
        if self.cpu_workers + self.gpu_workers == 0:
            raise SimulationError("need at least one worker")


class Worker:
    """A worker as the policy hooks see it (sim.py:39-46): id (CPU workers
    first), device, memory node, name, the time it next idles, busy flag.
    The device simulator keeps the same state per worker in its scratch."""

    def __init__(self, wid: int, device: str, name: str):
        self.id = wid
        self.device = device
        self.name = name
        self.mem_node = DEVICE if device == GPU else HOST
        self.free_time = 0.0
        self.busy = False


@dataclass(frozen=True)
class TraceEvent:
    """sim.py:49-54"""
    time: float
    kind: str
    subject: str
    resource: str


@dataclass
class Trace:
    """sim.py:57-65"""
    events: List[TraceEvent]
    makespan: float
    transfer_count: int
    transfer_bytes: int
    busy_ms: Dict[str, float]
    kernels_per_device: Dict[str, int]
    policy: str = ""


def _policy_id(policy) -> int:
    pid = getattr(policy, "native_id", None)
    # a subclass that overrides a hook is a custom policy: the device runs
    # only the built-in state machines
    if pid is not None:
        from . import policies as _p
        base = (_p.EagerPolicy, _p.DmdaPolicy, _p.GraphPartitionPolicy)[pid]
        cls = type(policy)
        if any(getattr(cls, h, None) is not getattr(base, h, None)
               for h in ("on_ready", "next_for_worker", "_estimate")):
            pid = None
    if pid is None:
        raise SimulationError(
            f"policy {type(policy).__name__} not supported by native backend "
            "(built-in eager/dmda/gp only)")
    return pid


def _check_graph(graph: TaskGraph) -> None:
    """sim.py:72-78"""
    problems = validate(graph)
    if problems:
        raise SimulationError(f"invalid graph: {problems[0]}")
    for nid in graph.kernel_ids():
        node = graph.nodes[nid]
        if node.weight_cpu == 0 and node.weight_gpu == 0:
            raise SimulationError(f"kernel {nid} has no weights; attach a cost model")


def _pin_array(graphs: Sequence[TaskGraph], policies) -> Optional[torch.Tensor]:
    """Per-node pin bytes (1 = GPU). Every non-root kernel must be pinned: the
    reference's on_ready looks the kernel up in the pin map and raises
    KeyError for a missing one (policies.py:92-93); the root is never queued."""
    pins = []
    for g, p in zip(graphs, policies):
        ids = g.csr().host.ids
        pm = p.pin_map
        root = g.root
        missing = [int(i) for i in ids if int(i) != root and int(i) not in pm]
        if missing:
            raise KeyError(missing[0])
        pins.append(np.fromiter((1 if int(i) != root and pm[int(i)] == GPU else 0 for i in ids),
                                dtype=np.int8, count=len(ids)))
    return torch.from_numpy(np.concatenate(pins)).to(_native.device())


def _worker_names(machine: MachineModel) -> List[str]:
    return ([f"cpu{i}" for i in range(machine.cpu_workers)]
            + [f"gpu{i}" for i in range(machine.gpu_workers)])


def _resource_ranks(names: List[str]) -> List[int]:
    """rank[resource + 1] of every resource name ("bus" = -1) in string order."""
    allr = ["bus"] + names
    order = sorted(range(len(allr)), key=lambda i: allr[i])
    rank = [0] * len(allr)
    for r, i in enumerate(order):
        rank[i] = r
    return rank


def _events_to_trace(graph: TaskGraph, raw: np.ndarray, names: List[str]) -> List[TraceEvent]:
    """Python events of device records already in the reference's order
    (hs_trace_sort: sim.py:200-201 — time, kind, subject as a string,
    resource as a string)."""
    ids = graph.csr().host.ids
    out = []
    for rec in raw:
        kind = _KIND_NAMES[rec["kind"]]
        a, b = int(rec["a"]), int(rec["b"])
        if rec["kind"] >= 2:
            subject, resource = str(int(ids[a])), names[int(rec["resource"])]
        else:
            subject = f"d{int(ids[a])}.{int(ids[b])}" if b >= 0 else f"d{int(ids[a])}"
            resource = "bus"
        out.append(TraceEvent(float(rec["time"]), kind, subject, resource))
    return out


def _run(graphs: Sequence[TaskGraph], policies, machine: MachineModel, events: bool):
    pid = _policy_id(policies[0])
    batch = DagBatch([g.csr().host for g in graphs])
    pin = _pin_array(graphs, policies) if pid == 2 else None
    out = _native.simulate_batch(batch, pid, pin, machine.cpu_workers, machine.gpu_workers,
                                 events=events)
    host = {k: v.cpu().numpy() for k, v in out.items()}
    if (host["status"] != 0).any():
        raise AssertionError("simulation deadlocked on a valid DAG (bug)")
    return batch, host, out


def simulate(graph: TaskGraph, policy, machine: Optional[MachineModel] = None,
             seed: int = 0) -> Trace:
    """One simulation with its full event trace (sim.py:68-204)."""
    machine = machine or MachineModel()
    _policy_id(policy)
    _check_graph(graph)
    batch, h, d = _run([graph], [policy], machine, events=True)
    names = _worker_names(machine)
    cnt = int(h["ev_count"][0])
    isz = _native.EVENT_DTYPE.itemsize
    off = int(h["ev_off"][0])
    ev_dev = d["events"][off * isz:(off + cnt) * isz]
    dev = ev_dev.device
    ids = torch.from_numpy(np.ascontiguousarray(graph.csr().host.ids, dtype=np.int64)).to(dev)
    rank = torch.tensor(_resource_ranks(names), dtype=torch.int32, device=dev)
    perm = _native.trace_sort(ev_dev, cnt, ids, rank)
    raw = h["events"].view(_native.EVENT_DTYPE)[off:off + cnt][perm.cpu().numpy()]
    events = _events_to_trace(graph, raw, names)
    tr = Trace(events, float(h["makespan"][0]), int(h["transfer_count"][0]),
               int(h["transfer_bytes"][0]),
               {CPU: float(h["busy"][0, 0]), GPU: float(h["busy"][0, 1])},
               {CPU: int(h["kpd"][0, 0]), GPU: int(h["kpd"][0, 1])},
               policy=getattr(policy, "name", ""))
    # the device buffer and order behind the events: metrics() reduces it
    # on the device while the events are unchanged
    tr._device = (ev_dev, perm, cnt, graph.csr().n, machine.cpu_workers, events)
    return tr


@dataclass
class BatchResult:
    """Aggregates of a batch of simulations (no event traces)."""
    makespan: np.ndarray
    transfer_count: np.ndarray
    transfer_bytes: np.ndarray
    busy_ms: np.ndarray            # [B, 2] (CPU, GPU)
    kernels_per_device: np.ndarray  # [B, 2]


def simulate_batch(graphs: Sequence[TaskGraph], policies, machine: Optional[MachineModel] = None,
                   validate_graphs: bool = True) -> BatchResult:
    """Many independent simulations in one device launch (config 5).

    ``policies`` holds one policy per graph, all of the same built-in type.
    """
    machine = machine or MachineModel()
    if len(graphs) != len(policies):
        raise SimulationError("need one policy per graph")
    if not graphs:
        z = np.zeros(0)
        return BatchResult(z, z.astype(np.int64), z.astype(np.int64), z.reshape(0, 2),
                           z.reshape(0, 2).astype(np.int64))
    ids = {_policy_id(p) for p in policies}
    if len(ids) != 1:
        raise SimulationError("a batch must use a single policy type")
    if validate_graphs:
        for g in graphs:
            _check_graph(g)
    _, h, _ = _run(graphs, policies, machine, events=False)
    return BatchResult(h["makespan"], h["transfer_count"], h["transfer_bytes"], h["busy"],
                       h["kpd"])


def metrics(trace: Trace) -> Dict[str, object]:
    """Summary recomputed from the events (sim.py:207-236).

    A trace from simulate() keeps its device event buffer: the summary is
    reduced there (hs_trace_metrics, busy times summed in event order as the
    reference does). Traces built or edited on the host take the host loop.
    """
    dv = getattr(trace, "_device", None)
    if dv is not None and dv[5] is trace.events and len(trace.events) == dv[2]:
        ev, perm, cnt, n_nodes, cpu_workers, _ = dv
        mk, nx, b0, b1, k0, k1 = _native.trace_metrics(ev, perm, cnt, n_nodes, cpu_workers)
        busy = {CPU: b0, GPU: b1}
        return {
            "makespan": mk,
            "transfer_count": int(nx),
            "transfer_bytes": trace.transfer_bytes,
            "busy_ms": busy,
            "busy_fraction": {d: (busy[d] / mk if mk else 0.0) for d in busy},
            "kernels_per_device": {CPU: int(k0), GPU: int(k1)},
        }
    starts: Dict[Tuple[str, str], float] = {}
    busy = {CPU: 0.0, GPU: 0.0}
    counts = {CPU: 0, GPU: 0}
    n_xfers = 0
    makespan = 0.0
    for e in trace.events:
        if e.kind == "kernel_start":
            starts[(e.subject, e.resource)] = e.time
        elif e.kind == "kernel_end":
            key = (e.subject, e.resource)
            if key not in starts:
                raise SimulationError(f"kernel_end without start for {key}")
            dev = CPU if e.resource.startswith("cpu") else GPU
            busy[dev] += e.time - starts.pop(key)
            counts[dev] += 1
            makespan = max(makespan, e.time)
        elif e.kind == "xfer_end":
            n_xfers += 1
    if starts:
        raise SimulationError(f"kernel_start without end for {sorted(starts)}")
    return {
        "makespan": makespan,
        "transfer_count": n_xfers,
        "transfer_bytes": trace.transfer_bytes,
        "busy_ms": busy,
        "busy_fraction": {d: (busy[d] / makespan if makespan else 0.0) for d in busy},
        "kernels_per_device": counts,
    }


def critical_path_lower_bound(graph: TaskGraph) -> float:
    """Longest path with each kernel's faster device time (sim.py:239-247), on device (K7)."""
    if not graph.nodes:
        return 0.0
    try:
        _, _, cp, _ = _native.levels(graph.csr(), mode=0)
    except _native.NativeError as exc:
        if "cycle" in exc.message:
            topological_order(graph)  # raises the reference's CycleError(min stuck id)
        raise
    return cp


def trace_csv(trace: Trace) -> str:
    """sim.py:250-255"""
    out = io.StringIO()
    out.write("time,kind,subject,resource\n")
    for e in trace.events:
        out.write(f"{e.time!r},{e.kind},{e.subject},{e.resource}\n")
    return out.getvalue()


def annotated_dot(graph: TaskGraph, trace: Trace) -> str:
    """DOT with each kernel's device and start/end times from a finished
    trace (sim.py:319-331); canonical emission as graphio.emit_dot."""
    from .graphio import emit_dot
    info: Dict[int, Dict[str, str]] = {}
    for e in trace.events:
        if e.kind in ("kernel_start", "kernel_end"):
            kid = int(e.subject)
            d = info.setdefault(kid, {})
            d["device"] = CPU if e.resource.startswith("cpu") else GPU
            d["start" if e.kind == "kernel_start" else "end"] = repr(e.time)
    node_extra = {kid: [("device", d["device"]), ("start", d["start"]), ("end", d["end"])]
                  for kid, d in info.items()}
    return emit_dot(graph, node_extra=node_extra)


@dataclass
class CompareRow:
    """sim.py:258-266"""
    policy: str
    mean_makespan: float
    sd_makespan: float
    mean_transfers: float
    sd_transfers: float
    mean_transfer_bytes: float
    size: Optional[int] = None


def compare(policy_names: Sequence[str], graph_factory: Callable[[int], TaskGraph],
            machine: Optional[MachineModel] = None, iterations: int = 1, seed: int = 0,
            policy_builder: Optional[Callable[[str, TaskGraph], object]] = None
            ) -> List[CompareRow]:
    """Mean/sd of makespan and transfers per policy over iterations (sim.py:269-306).

    As the reference: for every policy, iteration i calls graph_factory(seed
    + i), builds the policy on that graph and simulates it; the calls happen
    in the reference's order (policy-major), so stateful factories and
    builders see the same sequence. The simulations of a policy then run as
    one device batch (and the default gp builds as one batched partition).
    A gen.RandomDagFactory is generated on the device instead (identical
    graphs, see _compare_generated).
    """
    if iterations < 1:
        raise SimulationError("iterations must be >= 1")
    if policy_builder is None and hasattr(graph_factory, "batch"):
        return _compare_generated(policy_names, graph_factory, machine or MachineModel(),
                                  iterations, seed)
    batched_gp = policy_builder is None
    if policy_builder is None:
        from .policies import build_policy
        policy_builder = lambda name, g: build_policy(name, g)  # noqa: E731
    machine = machine or MachineModel()
    rows: List[CompareRow] = []
    for name in policy_names:
        graphs, policies = [], []
        gp_batch = name == "gp" and batched_gp
        for i in range(iterations):
            g = graph_factory(seed + i)
            if not gp_batch:
                policies.append(policy_builder(name, g))
            _check_graph(g)  # simulate's validation (sim.py:72-78)
            graphs.append(g)
        if gp_batch:  # all gp decisions in one device launch
            from .policies import gp_build_batch
            policies = gp_build_batch(graphs)
        res = simulate_batch(graphs, policies, machine, validate_graphs=False)
        makespans = [float(x) for x in res.makespan]
        transfers = [float(x) for x in res.transfer_count]
        t_bytes = [float(x) for x in res.transfer_bytes]
        rows.append(CompareRow(
            policy=name,
            mean_makespan=statistics.fmean(makespans),
            sd_makespan=statistics.stdev(makespans) if len(makespans) > 1 else 0.0,
            mean_transfers=statistics.fmean(transfers),
            sd_transfers=statistics.stdev(transfers) if len(transfers) > 1 else 0.0,
            mean_transfer_bytes=statistics.fmean(t_bytes),
        ))
    return rows


def _generated_results(policy_names, factory, machine, seeds) -> dict:
    """Per-iteration (makespan, transfers, transfer bytes) of every policy over
    the factory's graphs for `seeds`, built and simulated on the device."""
    from .policies import DMDA_ID, EAGER_ID, GP_ID, POLICY_NAMES, gp_pins_batch
    ids = {"eager": EAGER_ID, "dmda": DMDA_ID, "gp": GP_ID}
    for name in policy_names:
        if name not in ids:  # build_policy's error (policies.py:111-120)
            raise ValueError(f"unknown policy {name!r}; expected one of {POLICY_NAMES}")
    out = {}
    if not len(seeds):
        return {name: (np.zeros(0), np.zeros(0), np.zeros(0)) for name in policy_names}
    batch = factory.batch(list(seeds))
    for name in policy_names:
        pin = gp_pins_batch(batch) if name == "gp" else None
        res = _native.simulate_batch(batch, ids[name], pin, machine.cpu_workers,
                                     machine.gpu_workers, events=False)
        h = {k: v.cpu().numpy() for k, v in res.items()}
        if (h["status"] != 0).any():
            raise AssertionError("simulation deadlocked on a valid DAG (bug)")
        out[name] = (h["makespan"].astype(np.float64), h["transfer_count"].astype(np.float64),
                     h["transfer_bytes"].astype(np.float64))
    return out


def _row(name, makespans, transfers, t_bytes) -> CompareRow:
    """sim.py:296-306: fmean / stdev over the iterations in seed order."""
    makespans, transfers, t_bytes = ([float(x) for x in a] for a in (makespans, transfers, t_bytes))
    return CompareRow(
        policy=name,
        mean_makespan=statistics.fmean(makespans),
        sd_makespan=statistics.stdev(makespans) if len(makespans) > 1 else 0.0,
        mean_transfers=statistics.fmean(transfers),
        sd_transfers=statistics.stdev(transfers) if len(transfers) > 1 else 0.0,
        mean_transfer_bytes=statistics.fmean(t_bytes),
    )


def _compare_generated(policy_names, factory, machine, iterations, seed) -> List[CompareRow]:
    """compare() over a generator factory (gen.RandomDagFactory): every
    iteration's graph built on the device at once (csrc/rgen.cu, identical to
    the factory's own graphs), gp pins from one batched partition launch, one
    DES launch per policy. Same rows as the object path."""
    res = _generated_results(policy_names, factory, machine, [seed + i for i in range(iterations)])
    return [_row(name, *res[name]) for name in policy_names]


def iteration_split(iterations: int, world: int, rank: int) -> range:
    """The iterations rank `rank` simulates: contiguous, sizes differing by at most one."""
    q, r = divmod(iterations, world)
    lo = rank * q + min(rank, r)
    return range(lo, lo + q + (1 if rank < r else 0))


def gather_rows(policy_names, local: dict, group=None) -> List[CompareRow]:
    """Every rank's per-iteration results (its iteration_split share) gathered in
    iteration order, then the reference's rows: identical on every rank and to
    one device running all iterations."""
    import torch.distributed as dist
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if world > 1:
        parts = [None] * world
        dist.all_gather_object(parts, {k: tuple(np.asarray(a) for a in v) for k, v in local.items()},
                               group=group)
    else:
        parts = [local]
    rows = []
    for name in policy_names:
        cols = [np.concatenate([p[name][c] for p in parts]) for c in range(3)]
        rows.append(_row(name, *cols))
    return rows


def compare_distributed(policy_names: Sequence[str], factory, machine: Optional[MachineModel] = None,
                        iterations: int = 1, seed: int = 0, group=None) -> List[CompareRow]:
    """compare() over a gen.RandomDagFactory with the iterations split across the
    ranks of torch.distributed (independent simulations, no
    inter-GPU traffic on the critical path): rank r generates and simulates its
    contiguous share of the seeds on its own GPU, then the small per-iteration
    arrays are all-gathered in seed order. Every rank returns the rows compare()
    returns on one GPU, bit for bit. Without a process group it is compare()."""
    import torch.distributed as dist
    if iterations < 1:
        raise SimulationError("iterations must be >= 1")
    machine = machine or MachineModel()
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    mine = iteration_split(iterations, world, rank)
    local = _generated_results(policy_names, factory, machine, [seed + i for i in mine])
    return gather_rows(policy_names, local, group)


def compare_csv(rows: Sequence[CompareRow]) -> str:
    """sim.py:309-316"""
    out = io.StringIO()
    out.write("policy,size,mean_makespan,sd_makespan,mean_transfers,sd_transfers\n")
    for r in sorted(rows, key=lambda r: (r.size if r.size is not None else -1, r.policy)):
        size = "" if r.size is None else str(r.size)
        out.write(f"{r.policy},{size},{r.mean_makespan!r},{r.sd_makespan!r},"
                  f"{r.mean_transfers!r},{r.sd_transfers!r}\n")
    return out.getvalue()
