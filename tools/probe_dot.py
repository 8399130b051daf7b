"""DOT ingestion timing on the config-2 DAG (100k tasks / 1M edges) as emit_dot
text: parse_dot_csr end to end (host bytes -> device CSR), its stages, the
device CSR checked against the generated one, and the oracle on a sample."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1502_07451_b200 import kway, _native
from paper_1502_07451_b200.graphio import parse_dot_csr


def dot_text(c, kind="MA", size=512):
    op = c.out_ptr.cpu().numpy(); od = c.out_dst.cpu().numpy()
    wc = c.w_cpu.cpu().numpy().tolist(); wg = c.w_gpu.cpu().numpy().tolist()
    wx = c.w_xfer.cpu().numpy().tolist(); nb = c.bytes.cpu().numpy().tolist()
    lines = ["digraph cfg2 {"]
    for i in range(c.n):
        k, s = ("SOURCE", 0) if i == c.root else (kind, size)
        lines.append(f"  n{i} [kind={k}, size={s}, weight_cpu={wc[i]!r}, weight_gpu={wg[i]!r}];")
    src = np.repeat(np.arange(c.n), np.diff(op)).tolist(); dst = od.tolist()
    for j in range(c.m):
        lines.append(f"  n{src[j]} -> n{dst[j]} [bytes={nb[j]}, weight_xfer={wx[j]!r}];")
    lines.append("}")
    return "\n".join(lines) + "\n"


c2 = kway.layered_dag(100_000, 1_000_000, seed=0)
t0 = time.perf_counter(); text = dot_text(c2); data = text.encode(); t1 = time.perf_counter()
print(f"text {len(data)/1e6:.1f} MB, {text.count(chr(10))} lines, built in {t1-t0:.2f} s")
for _ in range(2):
    csr = parse_dot_csr(data)
torch.cuda.synchronize()
reps = 5
t0 = time.perf_counter()
for _ in range(reps):
    csr = parse_dot_csr(data)
torch.cuda.synchronize()
e2e = (time.perf_counter() - t0) / reps
print(f"parse_dot_csr e2e {e2e*1e3:.2f} ms = {len(data)/e2e/1e9:.2f} GB/s")
ok = (csr.n == c2.n and csr.m == c2.m and torch.equal(csr.out_dst, c2.out_dst)
      and torch.equal(csr.out_ptr, c2.out_ptr) and torch.equal(csr.w_xfer, c2.w_xfer)
      and torch.equal(csr.w_gpu, c2.w_gpu) and torch.equal(csr.w_cpu, c2.w_cpu))
print("csr identical to the generated DAG:", ok)
# device part alone: text already in HBM
dev_text = torch.frombuffer(bytearray(data), dtype=torch.uint8).cuda()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for it in range(3):
    torch.cuda.synchronize(); a.record()
    info, hd = _native.dot_parse_device(dev_text, len(data)); r = hd.csr()
    b.record(); torch.cuda.synchronize(); hd.close()
print(f"device parse + csr (text resident) {a.elapsed_time(b):.2f} ms = {len(data)/a.elapsed_time(b)/1e6:.2f} GB/s")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import dot_oracle as D
lines = text.split("\n")
sample = "\n".join(lines[:20001]) + "\n}\n"
t0 = time.perf_counter(); D.parse(sample); dt = time.perf_counter() - t0
print(f"oracle {len(sample)/1e6:.2f} MB in {dt:.2f} s = {len(sample)/dt/1e6:.3f} MB/s")
