import sys, torch
sys.path.insert(0, ".")
from paper_1502_07451_b200 import kway
c2 = kway.layered_dag(100_000, 1_000_000, seed=0)
ew, nw = kway.integer_weights(c2.w_xfer), kway.integer_weights(c2.w_gpu)
r = kway.partition_kway(kway.symmetrize(c2, ew, nw), 8, tol=0.03)
parts = kway.kernel_to_node_parts(c2, r.part).unsqueeze(0).repeat(64, 1).contiguous()
nw64 = nw.to(torch.int64)
e = kway.evaluate_batch(c2, parts, 8, nw64); torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(5): e = kway.evaluate_batch(c2, parts, 8, nw64)
b.record(); torch.cuda.synchronize()
print("evaluate 64 assignments ms", a.elapsed_time(b) / 5, int(e["xfer_count"][0]), int(e["xfer_bytes"][0]), int(e["cut_bytes"][0]))
