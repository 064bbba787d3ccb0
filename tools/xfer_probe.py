"""Host<->device transfer and allocation costs for the C4 matrix (8.6 GB), pinned host memory."""
import ctypes
import time

import torch

n = 32768
nbytes = n * n * 8
h = torch.empty(n * n, dtype=torch.float64, pin_memory=True)
h.fill_(1.0)
d = torch.empty(n * n, dtype=torch.float64, device="cuda")
for name, fn in [("H2D", lambda: d.copy_(h, non_blocking=True)), ("D2H", lambda: h.copy_(d, non_blocking=True))]:
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"{name}: {ms:.1f} ms = {nbytes / ms / 1e6:.1f} GB/s")
rt = ctypes.CDLL("libcudart.so") if False else None
del d
torch.cuda.empty_cache()
cudart = ctypes.CDLL(torch.cuda.__file__.replace("cuda/__init__.py", "lib/libcudart.so.12")) if False else None
# cudaMalloc / cudaFree timing through the library's own runtime (statically linked): use torch's raw allocator path
torch.cuda.synchronize()
t0 = time.perf_counter()
x = torch.cuda.caching_allocator_alloc(nbytes)
torch.cuda.synchronize()
t1 = time.perf_counter()
torch.cuda.caching_allocator_delete(x)
torch.cuda.empty_cache()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"cudaMalloc {nbytes / 1e9:.1f} GB: {(t1 - t0) * 1e3:.1f} ms, free: {(t2 - t1) * 1e3:.1f} ms")
