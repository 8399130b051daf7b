import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1502_07451_b200.cholesky import TiledCholesky, spd_matrix
for n in [int(x) for x in sys.argv[1:]]:
    A = spd_matrix(n, 0)
    c = TiledCholesky(n)
    c.load(A); c.run(); torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        c.load(A); torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); c.run(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    L = c.result()
    res = ((L @ L.T - A).abs().max() / A.abs().max()).item()
    t = min(ts)
    print(f"n={n} T={n//512} ms={t:.2f} GFLOP/s={c.flops/t/1e6:.0f} ({100*c.flops/t/1e9/37.0:.1f}% of 37 TF) resid={res:.2e}", flush=True)
    del A, c, L; torch.cuda.empty_cache()
