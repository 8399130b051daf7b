"""Time/quality sweep of partitioner knobs on one 10M DAG (env vars set per run)."""
import os, sys, subprocess, json
here = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = r'''
import sys, torch, json
sys.path.insert(0, %r)
from paper_1502_07451_b200 import kway
csr = kway.layered_dag(10_000_000, 100_000_000, 0)
ew, nw = kway.integer_weights(csr.w_xfer), kway.integer_weights(csr.w_gpu)
ug = kway.symmetrize(csr, ew, nw, kway.in_order(csr, ew))
for _ in range(2): r = kway.partition_kway(ug, 8, seed=0)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(3): r = kway.partition_kway(ug, 8, seed=0)
b.record(); torch.cuda.synchronize()
for _ in range(2): kway.symmetrize(csr, ew, nw, kway.in_order(csr, ew))
ew_in = kway.in_order(csr, ew)
torch.cuda.synchronize()
c, d = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
c.record()
for _ in range(3): kway.symmetrize(csr, ew, nw, ew_in)
d.record(); torch.cuda.synchronize()
print(json.dumps({"ms": a.elapsed_time(b) / 3, "sym_ms": c.elapsed_time(d) / 3, "cut": r.cut, "frac": r.cut / (ug.nnz // 2 * 19), "levels": r.levels,
                  "coarsest": r.coarsest, "feasible": r.feasible, "passes": r.refine_passes}))
''' % here
for spec in sys.argv[1:]:
    env = dict(os.environ)
    for kv in spec.split(","):
        k, v = kv.split("=")
        env[k] = v
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    print(spec, out.stdout.strip() or out.stderr[-500:], flush=True)
