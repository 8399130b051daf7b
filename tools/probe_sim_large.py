"""simulate() on the config-1 and config-3 Cholesky DAGs (120 / 45,760 tasks): full device traces."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1502_07451_b200 as H
from paper_1502_07451_b200.gen import cholesky_dag
from paper_1502_07451_b200.policies import GraphPartitionPolicy
from paper_1502_07451_b200.sim import critical_path_lower_bound, trace_csv

# per-tile timings (512x512 fp64): GPU from the K9 executor's measured items,
# CPU from host LAPACK at ~47 GFLOP/s; transfer over PCIe-class 50 GB/s
CAL = """kind,size,time_cpu_ms,time_gpu_ms
POTRF,512,0.95,1.5
TRSM,512,2.9,0.046
SYRK,512,2.9,0.05
GEMM,512,5.7,0.091
[transfer]
latency_ms,bandwidth_bytes_per_ms
0.01,50000000
"""
model = H.load_calibration(CAL)
for T in (8, 16, 64):
    g = cholesky_dag(T, model=model)
    t = H.workload_ratio(g)
    t0 = time.perf_counter()
    for name in ("eager", "dmda", "gp"):
        if name == "gp" and T > 16:
            continue  # the reference's 2-way FM (n^2.4) does not reach 45k tasks
        pol = H.build_policy(name, g, t)
        a = time.perf_counter()
        tr = H.simulate(g, pol, H.MachineModel(3, 1))
        b = time.perf_counter()
        n_x = tr.transfer_count
        print(f"T={T} tasks={len(g.kernel_ids())} {name}: makespan {tr.makespan:.3f} ms, "
              f"transfers {n_x}, events {len(tr.events)} (= 4x{len(g.kernel_ids())} + 2x{n_x}: "
              f"{len(tr.events) == 4 * len(g.kernel_ids()) + 2 * n_x}), cp {critical_path_lower_bound(g):.3f}, "
              f"{(b - a) * 1e3:.1f} ms wall", flush=True)
    if T <= 16:
        csv = trace_csv(tr)
        print("  trace_csv lines", csv.count("\n"))
