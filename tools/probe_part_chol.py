import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1502_07451_b200.cholesky import (PartitionedCholesky, owner_cyclic, owner_partition, spd_matrix,
                                             task_table, transfer_count, TASK_FLOPS_B3)
n = int(sys.argv[1])
A = spd_matrix(n, 0)
tb = task_table(n // 512)
kind = tb.kind.cpu().numpy()
w = np.array([TASK_FLOPS_B3[k] for k in kind])
for P in [int(x) for x in sys.argv[2:]]:
    for name, fn in (("cyclic", owner_cyclic), ("partition", owner_partition)):
        own = fn(tb, P)
        loads = np.bincount(own, weights=w, minlength=P)
        pc = PartitionedCholesky(n, own, P, mode="loopback")
        pc.load(A); pc.run(); torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        pc.load(A); torch.cuda.synchronize()
        a.record(); pc.run(); b.record(); torch.cuda.synchronize()
        ms = a.elapsed_time(b)
        print(f"n={n} P={P} {name:9s} ms={ms:8.1f} GF/s={n**3/3/ms/1e6:7.0f} transfers={transfer_count(tb, own):6d} "
              f"copies={sum(pc.copies):6d} load_imb={loads.max()/loads.mean():.3f}", flush=True)
        del pc; torch.cuda.empty_cache()
