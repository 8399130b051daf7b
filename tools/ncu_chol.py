import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1502_07451_b200.cholesky import TiledCholesky, spd_matrix
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
A = spd_matrix(n, 0)
c = TiledCholesky(n)
c.load(A); c.run(); torch.cuda.synchronize()
print("ok")
