"""Pageable H2D of a Python bytes object vs registering it in place
(cudaHostRegister, read-only) for the copy."""
import ctypes, sys, time, warnings
import torch
n = 76 << 20
data = bytes(bytearray(n))
dev = torch.empty(n, dtype=torch.uint8, device="cuda")
warnings.simplefilter("ignore")
host = torch.frombuffer(data, dtype=torch.uint8)
cud = torch.cuda.cudart()
addr = ctypes.cast(ctypes.c_char_p(data), ctypes.c_void_p).value
for mode in ("pageable", "register", "pageable", "register"):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if mode == "register":
        r = cud.cudaHostRegister(addr, n, 8)
        t1 = time.perf_counter()
        dev.copy_(host)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        cud.cudaHostUnregister(addr)
        t3 = time.perf_counter()
        print(mode, r, f"register {1e3*(t1-t0):.2f} copy {1e3*(t2-t1):.2f} unregister {1e3*(t3-t2):.2f} total {1e3*(t3-t0):.2f} ms")
    else:
        dev.copy_(host)
        torch.cuda.synchronize()
        print(mode, f"{1e3*(time.perf_counter()-t0):.2f} ms")
