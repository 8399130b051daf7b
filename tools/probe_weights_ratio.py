import sys; sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import test_gpu_kway_weights as T, torch
from paper_1502_07451_b200 import kway
for k in (2, 8, 16, 32):
    csr = kway.layered_dag(100_000, 1_000_000, 0); ew, nw = T._random_weights(csr, 1, 100, seed=k)
    r = kway.partition_kway(kway.symmetrize(csr, ew, nw), k, tol=0.03, seed=3)
    print("cfg2 U k", k, r.cut / T._band_cut(csr, k, ew, nw), r.max_deviation)
for tiles, k in ((16, 4), (32, 8), (64, 8)):
    g = T.cholesky_dag(tiles, 512, T.load_calibration(T.CHOL_CSV)); csr = g.csr()
    ew = kway.integer_weights(csr.w_xfer); nw = kway.integer_weights(csr.w_gpu)
    r = kway.partition_dag(csr, k, tol=0.03); print("chol", tiles, k, r.cut / T._band_cut(csr, k, ew, nw), r.levels)
