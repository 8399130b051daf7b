"""One config-4 partition step (K1 + K3-K6) inside a cudaProfilerStart/Stop window,
after two warm-up steps: run under `ncu --profile-from-start off` for its launch list,
or plain for the step's wall/device time."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1502_07451_b200 import kway
csr = kway.layered_dag(10_000_000, 100_000_000, 0)
ew, nw = kway.integer_weights(csr.w_xfer), kway.integer_weights(csr.w_gpu)
ew_in = kway.in_order(csr, ew)


def step():
    return kway.partition_kway(kway.symmetrize(csr, ew, nw, ew_in), 8, tol=0.03, seed=0)


for _ in range(2):
    step()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.cudart().cudaProfilerStart()
t0 = time.perf_counter()
a.record()
r = step()
b.record()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print(f"step device {a.elapsed_time(b):.3f} ms wall {(time.perf_counter() - t0) * 1e3:.3f} ms cut {r.cut}")
