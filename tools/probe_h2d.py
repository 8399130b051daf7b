"""H2D/D2H bandwidth of pinned copies on this box (sizes of the e2e arrays)."""
import torch
dev = torch.device("cuda")
for mb in (40, 400, 920):
    h = torch.empty(mb << 20, dtype=torch.uint8).pin_memory()
    d = torch.empty_like(h, device=dev)
    for _ in range(2):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); d.copy_(h, non_blocking=True); b.record(); torch.cuda.synchronize()
    t = a.elapsed_time(b)
    a.record(); h.copy_(d, non_blocking=True); b.record(); torch.cuda.synchronize()
    t2 = a.elapsed_time(b)
    print(f"{mb} MB: H2D {mb / 1024 / t * 1e3:.1f} GiB/s ({t:.2f} ms), D2H {mb / 1024 / t2 * 1e3:.1f} GiB/s")
    # .to() of a pinned tensor
    a.record(); x = h.to(dev, non_blocking=True); b.record(); torch.cuda.synchronize()
    print(f"   .to(): {a.elapsed_time(b):.2f} ms")
