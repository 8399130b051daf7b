import time, sys, torch
sys.path.insert(0, ".")
from paper_1502_07451_b200 import kway, _native
for (n, m, k) in [(100_000, 1_000_000, 8), (10_000_000, 100_000_000, 8)]:
    t0 = time.time()
    csr = kway.layered_dag(n, m, 0)
    torch.cuda.synchronize(); t1 = time.time()
    ew = kway.integer_weights(csr.w_xfer); nw = kway.integer_weights(csr.w_gpu)
    torch.cuda.synchronize()
    for rep in range(3):
        ts = time.time()
        ug = kway.symmetrize(csr, ew, nw)
        torch.cuda.synchronize(); t2 = time.time()
        r = kway.partition_kway(ug, k, seed=0)
        torch.cuda.synchronize(); t3 = time.time()
        print(f"n={n} m={m} gen={t1-t0:.3f}s sym={1e3*(t2-ts):.1f}ms part={1e3*(t3-t2):.1f}ms cut={r.cut} "
              f"frac={r.cut/ (ug.nnz//2 * int(ew[0])):.4f} levels={r.levels} coarsest={r.coarsest} dev={r.max_deviation:.4f} "
              f"feas={r.feasible} passes={r.refine_passes}", flush=True)
    del ug, csr
    torch.cuda.empty_cache()
