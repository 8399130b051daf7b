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
    st = torch.zeros(16, dtype=torch.int64, device="cuda")
    c.load(A); c.run(st); torch.cuda.synchronize()
    st = st.cpu().tolist()
    ghz = 1.965e6  # cycles per ms
    names = ["POTRF", "TRSM", "SYRK", "GEMM"]
    print("  per item us:", {names[i]: round(st[2*i] / max(1, st[2*i+1]) / ghz * 1e3, 1) for i in range(4)},
          "items:", {names[i]: st[2*i+1] for i in range(4)},
          "POTRF phases us/call:", [round(x / max(1, st[1]) / ghz * 1e3, 1) for x in st[8:11]],
          "diag A/B1/B2 us/call:", [round(x / max(1, st[1]) / ghz * 1e3, 1) for x in st[11:14]],
          "busy CTA-ms:", round(sum(st[0:8:2]) / ghz, 1), flush=True)
    L = c.result()
    res = ((L @ L.T - A).abs().max() / A.abs().max()).item()
    t = min(ts)
    print(f"n={n} T={n//512} ms={t:.2f} GFLOP/s={c.flops/t/1e6:.0f} ({100*c.flops/t/1e9/37.0:.1f}% of 37 TF) resid={res:.2e}", flush=True)
    del A, c, L; torch.cuda.empty_cache()
